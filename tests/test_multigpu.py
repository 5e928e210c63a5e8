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


def _two_rank_run(sc, steps, world=2):
    engs = [capi.gpu_engine(sc, capture=True, rank=r, world=world) for r in range(world)]
    pools = [e.pool_pointers() for e in engs]
    for r, e in enumerate(engs):
        for q in range(world):
            if q != r:
                e.set_peer_pools(q, pools[q])
    for e in engs:
        e.prepare()
    dist.step_same_process(engs, steps)
    return engs


@pytest.mark.gpu
@pytest.mark.parametrize("name,world", [("mpmc_e32", 2), ("mpmc_progressive_e16", 2),
                                        ("mpmc_e32_solid_periodic", 2), ("mpmc_s0_3dev", 3),
                                        ("c1_progressive", 2), ("mpmc_islands", 2),
                                        ("mpmc_e64", 2)])
def test_ranks_in_one_process_match_single_engine(built, name, world):
    import numpy as np
    from tests.compare import FIELDS
    make, steps = scenarios.ALL[name]
    sc = make()
    sc.devices = max(sc.devices, world)  # owners spread over the ranks
    single = capi.gpu_engine(sc, capture=True)
    single.step(steps)
    engs = _two_rank_run(sc, steps, world)
    ref_c = single.counters()
    for e in engs:
        c = e.counters()
        for k in ("iteration", "cell_updates", "suppressed_expansions", "tiles", "active_cells", "bytes"):
            assert c[k] == ref_c[k], (k, c[k], ref_c[k])
        assert e.creation_log() == single.creation_log()
        assert e.tiles() == single.tiles()
    for k in ("negative_populations", "psi_clamps", "zero_rho_forcings"):
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


def _proc_rank(rank, world, port, name, steps, q):
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
        stepper = dist.DistStepper(eng, td, 0)
        stepper.step(steps)
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
@pytest.mark.parametrize("name", ["mpmc_progressive_e16", "mpmc_e32"])
def test_two_processes_one_gpu_match_single_engine(built, name):
    """The DistStepper protocol across real processes (IPC-mapped peer pools,
    torch.distributed collectives): bit-identical to one engine."""
    import socket
    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    _, steps = scenarios.ALL[name]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_proc_rank, args=(r, 2, port, name, steps, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict((r, (m, b)) for r, m, b in (q.get(timeout=600) for _ in procs))
    for p in procs:
        p.join(120)
    for r in range(2):
        mine, bad = res[r]
        assert mine > 0 and not bad, (r, mine, bad)
