"""Multi-GPU path.

GPU: several ranks' engines in one process on one B200, attached to each
other's pools, must reproduce the single-engine (and oracle) state bit for bit
— the same fused kernels then read neighbour tiles from another rank's pool,
exactly as they do over NVLink on a multi-GPU box.

CPU: the host-side trigger merge across ranks over torch.distributed/gloo
(world size 2).
"""
import os

import numpy as np
import pytest

from paper_1510_03560_b200 import capi, dist
from tests import scenarios


def _gloo_worker(rank, world, port, q):
    import torch
    import torch.distributed as td
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    td.init_process_group("gloo", rank=rank, world_size=world)
    n = 37
    local = np.zeros(n, np.uint8)
    # rank r owns slots r, r+world, ...; only owners set bits
    for s in range(rank, n, world):
        local[s] = (s * 7 + 3) & 0x3F
    def allreduce_max(a):
        t = torch.from_numpy(a.copy())
        td.all_reduce(t, op=td.ReduceOp.MAX)
        return t.numpy()
    merged = dist.merge_triggers(local, allreduce_max)
    q.put((rank, merged.tolist()))
    td.destroy_process_group()


def test_trigger_merge_over_gloo_world2():
    import socket
    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(60)
    want = [(s * 7 + 3) & 0x3F for s in range(37)]
    assert res[0] == want and res[1] == want


def _attach(sc, world, storage="ab"):
    engs = [capi.gpu_engine(sc, capture=True, rank=r, world=world, storage=storage) for r in range(world)]
    pools = [e.pool_pointers() for e in engs]
    for r, e in enumerate(engs):
        for q in range(world):
            if q != r:
                e.set_peer_pools(q, pools[q])
    for e in engs:
        e.prepare()
    return engs


def _two_rank_run(sc, steps, world=2, protocol="device", storage="ab"):
    engs = _attach(sc, world, storage)
    if protocol == "device":  # plbm_gpu_step on every rank (device barriers + expansion)
        for chunk in (1, 2, steps - 3):
            dist.step_ranks_threaded(engs, chunk)
    else:                     # host-merge protocol
        dist.step_same_process(engs, steps)
    return engs


@pytest.mark.gpu
@pytest.mark.parametrize("protocol,storage", [("device", "ab"), ("host", "ab"), ("device", "aa")])
@pytest.mark.parametrize("name,world", [("mpmc_e32", 2), ("mpmc_progressive_e16", 2),
                                        ("mpmc_e32_solid_periodic", 2), ("mpmc_s0_3dev", 3),
                                        ("c1_progressive", 2), ("mpmc_islands", 2),
                                        ("mpmc_e64", 2), ("mpmc_channel_e16", 4)])
def test_ranks_in_one_process_match_single_engine(built, name, world, protocol, storage):
    """Several ranks' engines in one process on one GPU, attached to each
    other's pools: the device protocol (plbm_gpu_step with rank barriers and
    replicated device expansion, one host thread per rank) and the host-merge
    protocol reproduce one engine bit for bit, with A-B or A-A storage."""
    import numpy as np
    from tests.compare import FIELDS
    make, steps = scenarios.ALL[name]
    sc = make()
    if storage == "aa" and sc.tile_extent > 32 and sc.n_components > 2:
        pytest.skip("A-A storage needs tile_extent <= 32")
    sc.devices = max(sc.devices, world)  # owners spread over the ranks
    single = capi.gpu_engine(sc, capture=True)
    single.step(steps)
    engs = _two_rank_run(sc, steps, world, protocol, storage)
    ref_c = single.counters()
    for e in engs:
        c = e.counters()
        for k in ("iteration", "cell_updates", "suppressed_expansions", "tiles", "active_cells", "bytes"):
            assert c[k] == ref_c[k], (k, c[k], ref_c[k])
        assert e.creation_log() == single.creation_log()
        assert e.tiles() == single.tiles()
    for k in ("negative_populations", "psi_clamps", "zero_rho_forcings"):
        if protocol == "device":  # every rank reports the job-wide sums
            assert all(e.counters()[k] == ref_c[k] for e in engs), k
        else:                     # host-merge protocol: each rank its own tiles
            assert sum(e.counters()[k] for e in engs) == ref_c[k]
    owners = set()
    for coords, _, _ in single.tiles():
        r = engs[0].tile_rank(coords)
        owners.add(r)
        for comp in range(sc.n_components):
            for f in FIELDS:
                a = single.read_tile(coords, comp, f)
                b = engs[r].read_tile(coords, comp, f)
                assert np.array_equal(a.view(np.uint64), b.view(np.uint64)), (coords, comp, f)
    assert len(owners) == world  # the run really was split across ranks


def _proc_rank(rank, world, port, name, steps, q, protocol="device"):
    """One rank of a real multi-process run (gloo plumbing, CUDA IPC pools) on
    GPU 0, checked against a single-engine run of the same scenario."""
    try:
        import torch
        import torch.distributed as td
        from tests.compare import FIELDS
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        td.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        make, _ = scenarios.ALL[name]
        sc = make()
        sc.devices = max(sc.devices, world)
        eng = capi.gpu_engine(sc, capture=True, rank=rank, world=world)
        stepper = (dist.DistStepper if protocol == "device" else dist.HostMergeStepper)(eng, td, 0)
        stepper.step(1)
        stepper.step(steps - 1)
        eng.sync()
        single = capi.gpu_engine(sc, capture=True)
        single.step(steps)
        bad = []
        for k in ("iteration", "cell_updates", "suppressed_expansions", "tiles", "active_cells", "bytes"):
            if eng.counters()[k] != single.counters()[k]:
                bad.append(k)
        if eng.creation_log() != single.creation_log():
            bad.append("creation_log")
        mine = 0
        for coords, _, _ in single.tiles():
            if eng.tile_rank(coords) != rank:
                continue
            mine += 1
            for comp in range(sc.n_components):
                for f in FIELDS:
                    a = single.read_tile(coords, comp, f)
                    b = eng.read_tile(coords, comp, f)
                    if not np.array_equal(a.view(np.uint64), b.view(np.uint64)):
                        bad.append((coords, comp, f))
        td.barrier()
        td.destroy_process_group()
        q.put((rank, mine, bad[:5]))
    except Exception as ex:  # report instead of hanging the parent
        q.put((rank, -1, [repr(ex)]))


@pytest.mark.gpu
@pytest.mark.parametrize("protocol", ["device", "host"])
@pytest.mark.parametrize("name", ["mpmc_progressive_e16", "mpmc_e32"])
def test_two_processes_one_gpu_match_single_engine(built, name, protocol):
    """Both multi-rank protocols across real processes (IPC-mapped pools and
    sync blocks; device barriers, or torch.distributed collectives for the
    host merge): bit-identical to one engine."""
    import socket
    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    _, steps = scenarios.ALL[name]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_proc_rank, args=(r, 2, port, name, steps, q, protocol)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict((r, (m, b)) for r, m, b in (q.get(timeout=600) for _ in procs))
    for p in procs:
        p.join(120)
    for r in range(2):
        mine, bad = res[r]
        assert mine > 0 and not bad, (r, mine, bad)


@pytest.mark.gpu
@pytest.mark.parametrize("slow", [None, 0, 1])
@pytest.mark.parametrize("name", ["mpmc_progressive_e16", "mpmc_e32"])
def test_ranks_agree_on_engine_error(built, name, slow, monkeypatch):
    """EngineError on several ranks: a NaN poked into one rank's tile makes
    EVERY rank raise the same (iteration, tile, phase) as one engine — the
    device check merges the lowest error key of all ranks — with iteration and
    cell_updates not advanced anywhere."""
    from paper_1510_03560_b200.scenario import EngineError
    if slow is not None:  # one rank trails (ordering stress of the error merge)
        monkeypatch.setenv("PLBM_TEST_RANK_DELAY_US", f"{slow}:300")
    make, _ = scenarios.ALL[name]
    sc = make()
    sc.devices = max(sc.devices, 2)
    single = capi.gpu_engine(sc, capture=True)
    engs = _attach(sc, 2)
    single.step(3)
    dist.step_ranks_threaded(engs, 3)
    tiles = [t[0] for t in single.tiles()]
    coords = tiles[len(tiles) // 2]
    owner = engs[0].tile_rank(coords)
    E = sc.tile_extent
    local = (E // 2, E // 2 - 1, E // 2 + 1)
    single.poke_f(coords, 0, 7, local, float("nan"))
    engs[owner].poke_f(coords, 0, 7, local, float("nan"))
    want = None
    try:
        single.step(3)
    except EngineError as e:
        want = (e.iteration, tuple(e.tile), e.phase)
    assert want is not None
    errs = [None, None]

    def run(k):
        try:
            engs[k].step(3)
        except EngineError as ex:
            errs[k] = (ex.iteration, tuple(ex.tile), ex.phase)

    import threading
    th = [threading.Thread(target=run, args=(k,)) for k in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert errs[0] == want and errs[1] == want, (errs, want)
    for e in engs:
        for k in ("iteration", "cell_updates"):
            assert e.counters()[k] == single.counters()[k], k


@pytest.mark.gpu
@pytest.mark.parametrize("slow", [None, 0, 1])
@pytest.mark.parametrize("name", ["mpmc_progressive_e16", "c1_progressive"])
def test_ranks_overflow_to_host_expansion(built, name, slow, monkeypatch):
    """Several ranks, no launch headroom (PLBM_EXPAND_HEADROOM=0): every birth
    overflows the launched grid, the device check halts EVERY rank at the
    same step and each rank's host mirror expands from the merged trigger
    bytes the device kept — still bit-identical to one engine."""
    import numpy as np
    from tests.compare import FIELDS
    monkeypatch.setenv("PLBM_EXPAND_HEADROOM", "0")
    if slow is not None:  # one rank trails (ordering stress of the fallback)
        monkeypatch.setenv("PLBM_TEST_RANK_DELAY_US", f"{slow}:300")
    make, steps = scenarios.ALL[name]
    sc = make()
    sc.devices = max(sc.devices, 2)
    single = capi.gpu_engine(sc, capture=True)
    single.step(steps)
    engs = _two_rank_run(sc, steps, 2, "device")
    for e in engs:
        for k in ("iteration", "cell_updates", "suppressed_expansions", "tiles", "bytes"):
            assert e.counters()[k] == single.counters()[k], k
        assert e.creation_log() == single.creation_log()
    for coords, _, _ in single.tiles():
        r = engs[0].tile_rank(coords)
        for comp in range(sc.n_components):
            for f in FIELDS:
                a = single.read_tile(coords, comp, f)
                b = engs[r].read_tile(coords, comp, f)
                assert np.array_equal(a.view(np.uint64), b.view(np.uint64)), (coords, comp, f)


class _MockEngine:
    """Stands in for a GpuEngine on CPU: records the plumbing calls."""

    def __init__(self, rank):
        self.rank, self.opened, self.prepared, self.steps = rank, {}, False, []

    def ipc_handles(self):
        return bytes([self.rank]) * 192  # 3 x cudaIpcMemHandle_t

    def open_peer(self, r, h):
        self.opened[r] = h

    def prepare(self):
        self.prepared = True

    def step(self, n):
        self.steps.append(n)


def _plumbing_worker(rank, world, port, q):
    import torch.distributed as td
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    td.init_process_group("gloo", rank=rank, world_size=world)
    eng = _MockEngine(rank)
    stepper = dist.DistStepper(eng, td, 0)
    stepper.step(3)
    stepper.step(1)
    q.put((rank, sorted(eng.opened), [eng.opened[r][0] for r in sorted(eng.opened)], eng.prepared, eng.steps))
    td.destroy_process_group()


def test_device_protocol_plumbing_over_gloo_world2():
    """The N > 1 set-up of the device protocol on CPU (gloo, world size 2):
    every rank all-gathers the IPC handles, opens exactly its peers' handles,
    prepares, and then steps with plbm_gpu_step alone (no per-step host
    collective)."""
    import socket
    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_plumbing_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = {r: rest for r, *rest in (q.get(timeout=120) for _ in procs)}
    for p in procs:
        p.join(60)
    for r in range(2):
        peers, first_bytes, prepared, steps = res[r]
        assert peers == [1 - r] and first_bytes == [1 - r]
        assert prepared and steps == [3, 1]


@pytest.mark.gpu
def test_host_merge_protocol_ranks_agree_on_engine_error(built):
    """The host-merge protocol too: step_end merges the peers' error keys, so
    a NaN in one rank's tile gives both ranks the single engine's error."""
    import numpy as np
    from paper_1510_03560_b200.scenario import EngineError
    make, _ = scenarios.ALL["mpmc_e32"]
    sc = make()
    sc.devices = max(sc.devices, 2)
    single = capi.gpu_engine(sc, capture=True)
    engs = _attach(sc, 2)
    single.step(3)
    dist.step_same_process(engs, 3)
    tiles = [t[0] for t in single.tiles()]
    coords = tiles[len(tiles) // 2]
    owner = engs[0].tile_rank(coords)
    local = (16, 15, 17)
    single.poke_f(coords, 0, 7, local, float("nan"))
    engs[owner].poke_f(coords, 0, 7, local, float("nan"))
    want = None
    try:
        single.step(3)
    except EngineError as e:
        want = (e.iteration, tuple(e.tile), e.phase)
    assert want is not None
    errs = [None, None]
    for _ in range(3):
        for e in engs:
            e.step_main()
        for e in engs:
            e.sync()
        for e in engs:
            e.step_face()
        for e in engs:
            e.sync()
        merged = np.zeros(engs[0].trigger_bytes(), np.uint8)
        for e in engs:
            merged |= e.local_triggers()
        for k, e in enumerate(engs):
            try:
                e.step_end(merged)
            except EngineError as ex:
                errs[k] = (ex.iteration, tuple(ex.tile), ex.phase)
        if errs[0] or errs[1]:
            break
    assert errs[0] == want and errs[1] == want, (errs, want)


@pytest.mark.gpu
@pytest.mark.parametrize("slow", [0, 1])
@pytest.mark.parametrize("name", ["mpmc_progressive_e16", "mpmc_channel_e16", "c1_progressive"])
def test_ranks_with_one_rank_trailing(built, name, slow, monkeypatch):
    """Ordering stress of the device protocol: one rank spins 300 us on the
    device before every step, so its peer runs ahead into the barriers, the
    replicated expansion and the next step's pulls — still bit-identical."""
    import numpy as np
    from tests.compare import FIELDS
    monkeypatch.setenv("PLBM_TEST_RANK_DELAY_US", f"{slow}:300")
    make, steps = scenarios.ALL[name]
    sc = make()
    sc.devices = max(sc.devices, 2)
    single = capi.gpu_engine(sc, capture=True)
    single.step(steps)
    engs = _two_rank_run(sc, steps, 2, "device")
    for e in engs:
        for k in ("iteration", "cell_updates", "suppressed_expansions", "tiles", "bytes",
                  "negative_populations", "psi_clamps"):
            assert e.counters()[k] == single.counters()[k], k
        assert e.creation_log() == single.creation_log()
    for coords, _, _ in single.tiles():
        r = engs[0].tile_rank(coords)
        for comp in range(sc.n_components):
            for f in FIELDS:
                a = single.read_tile(coords, comp, f)
                b = engs[r].read_tile(coords, comp, f)
                assert np.array_equal(a.view(np.uint64), b.view(np.uint64)), (coords, comp, f)
