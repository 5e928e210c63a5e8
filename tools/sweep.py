#!/usr/bin/env python
"""Measurement sweeps on one B200 (results -> JSON lines on stdout).

    python tools/sweep.py c1 [--steps 500]
        BASELINE configs[0] (the reference's CPU scenario) on both engines in
        the same run: time to solution and identical creation log.
    python tools/sweep.py c5 [--n 256] [--steps 20]
        BASELINE configs[4] on one GPU: tile extent E in {16, 32} x components
        C in {1, 2, 3}, static full-domain MPMC (all tiles active), MLUPS per
        component of the whole step and of the fused kernel.
    python tools/sweep.py c4 [--steps 400] [--storage aa] [--static]
        BASELINE configs[3] on one GPU: MPMC release in the 3-D channel
        network (scenario.channel_network) at 1024x512x512, progressive; with
        --static also the static full mesh (8192 tiles: 174 GB of populations
        with two buffers, so --storage aa, one in-place buffer, to fit).
    python tools/sweep.py c3 [--n 512] [--steps 300]
        BASELINE configs[2], the paper's comparison: the same MPMC release run
        on the progressive mesh and on the static full-domain mesh for the
        same number of steps; wall time on the device, tiles over time.
    python tools/sweep.py ranks [--steps 30]
        The multi-rank device protocol on ONE GPU: the C2 bench workload split
        over 1, 2 and 4 ranks' engines in one process (one host thread per
        rank, attached to each other's pools, stepping with plbm_gpu_step's
        device barriers and replicated expansion); total MLUPS/comp against
        the single engine = the protocol's own cost (the ranks share one GPU,
        so this is not a scaling number).
    python tools/sweep.py placement [--steps 400]
        The paper's GPU-assignment study (simple vs optimized assign_device,
        PAPER.md Figures 13/16) on C4's channel network with 8 simulated
        devices in two NVLink islands of 4 (staged links between islands):
        placement runs inside the device-side expansion on one B200; reported
        per policy: tiles per device, the reference's modeled byte classes
        (record_exchange), and the cross-device face exchanges of the final
        mesh (what an 8-GPU run would move per step: 11 E^2 C doubles per
        face read by the kernels, 5 crossing populations + psi + the 5 of the
        face pass).
"""
import argparse
import json
import os
import sys
import time

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

from paper_1510_03560_b200 import capi  # noqa: E402
from paper_1510_03560_b200 import scenario as S  # noqa: E402

BYTES = 304


def timed(eng, steps, chunk=1):
    import torch
    stream = torch.cuda.ExternalStream(eng.stream())
    eng.reset_kernel_stats()
    eng.set_profiling(True)
    c0 = eng.counters()["cell_updates"]
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    done = 0
    while done < steps:
        k = min(chunk, steps - done)
        eng.step(k)
        done += k
    e1.record(stream)
    torch.cuda.synchronize()
    ks = eng.kernel_stats()
    eng.set_profiling(False)
    return e0.elapsed_time(e1), eng.counters()["cell_updates"] - c0, ks


def c5(a):
    for E in a.extents:
        for C in a.comps:
            sc = S.mpmc_release(n=a.n, extent=E, mode=S.MODE_STATIC, n_components=C)
            eng = capi.gpu_engine(sc, storage=a.storage)
            eng.step(a.warmup)
            ms, cells, ks = timed(eng, a.steps, chunk=a.steps)
            main = ks["main_cell_updates"] * C * BYTES / (ks["main_ms"] / 1e3) / 1e9
            print(json.dumps({
                "sweep": "c5", "E": E, "C": C, "domain": a.n, "tiles": eng.counters()["tiles"],
                "steps": a.steps, "ms_per_step": round(ms / a.steps, 4),
                "mlups_per_comp": round(cells * C / (ms / 1e3) / 1e6, 1),
                "k_main_ms": round(ks["main_ms"] / max(ks["main_launches"], 1), 4),
                "k_face_ms": round(ks["face_ms"] / max(ks["face_launches"], 1), 4),
                "k_main_algorithmic_GBs": round(main, 1)}), flush=True)
            eng.close()


def c3(a):
    out = {}
    for mode, name in ((S.MODE_PROGRESSIVE, "progressive"), (S.MODE_STATIC, "static")):
        sc = S.mpmc_release(n=a.n, extent=32, mode=mode, threshold=1e-9)
        eng = capi.gpu_engine(sc, storage=a.storage)
        series = []
        total_ms = 0.0
        for k0 in range(0, a.steps, a.every):
            ms, cells, _ = timed(eng, min(a.every, a.steps - k0), chunk=1 if mode == S.MODE_PROGRESSIVE else a.every)
            total_ms += ms
            series.append({"step": k0 + a.every, "tiles": eng.counters()["tiles"], "ms": round(ms, 3),
                           "pool_GB": round(eng.memory()["pool_mapped_bytes"] / 1e9, 2),
                           "map_ms": round(eng.memory()["map_host_ms"], 1),
                           "map_wait_ms": round(eng.memory()["map_wait_ms"], 1)})
        out[name] = {"total_ms": round(total_ms, 2), "final_tiles": eng.counters()["tiles"],
                     "cell_updates": eng.counters()["cell_updates"],
                     "pool_mapped_GB": round(eng.memory()["pool_mapped_bytes"] / 1e9, 2),
                     "pool_reserved_GB": round(eng.memory()["pool_reserved_bytes"] / 1e9, 2), "series": series}
        eng.close()
    out["speedup_progressive_vs_static"] = round(out["static"]["total_ms"] / out["progressive"]["total_ms"], 3)
    print(json.dumps({"sweep": "c3", "domain": a.n, "steps": a.steps, **out}), flush=True)


def c4(a):
    """BASELINE configs[3] on one GPU: the 3-D channel network at full size,
    progressive mesh, and with --static the static full domain on the same
    scenario (8192 tiles: 174 GB of A-B pool, 87 GB A-A)."""
    modes = [(S.MODE_PROGRESSIVE, "progressive")] + ([(S.MODE_STATIC, "static")] if a.static else [])
    out = {}
    for mode, name in modes:
        t0 = time.time()
        sc = S.mpmc_channel(nx=1024, ny=512, nz=512, extent=32, threshold=1e-9, mode=mode)
        eng = capi.gpu_engine(sc, storage=a.storage)
        if a.variant:
            eng.set_kernel_variant(a.variant)
        setup_s = time.time() - t0
        series, total_ms, cells = [], 0.0, 0
        for k0 in range(0, a.steps, a.every):
            ms, c, ks = timed(eng, min(a.every, a.steps - k0),
                              chunk=1 if mode == S.MODE_PROGRESSIVE else a.every)
            total_ms += ms
            cells += c
            series.append({"step": k0 + a.every, "tiles": eng.counters()["tiles"], "ms": round(ms, 3),
                           "mlups_per_comp": round(c * 2 / (ms / 1e3) / 1e6, 1),
                           "pool_GB": round(eng.memory()["pool_mapped_bytes"] / 1e9, 2),
                           "map_ms": round(eng.memory()["map_host_ms"], 1),
                           "map_wait_ms": round(eng.memory()["map_wait_ms"], 1)})
        out[name] = {"setup_s": round(setup_s, 2), "total_ms": round(total_ms, 2),
                     "pool_mapped_GB": round(eng.memory()["pool_mapped_bytes"] / 1e9, 2),
                     "pool_reserved_GB": round(eng.memory()["pool_reserved_bytes"] / 1e9, 2),
                     "final_tiles": eng.counters()["tiles"], "cell_updates": eng.counters()["cell_updates"],
                     "mlups_per_comp": round(cells * 2 / (total_ms / 1e3) / 1e6, 1), "series": series}
        fluid = round(1 - float(sc.geometry.mean()), 4)
        eng.close()
    line = {"sweep": "c4", "domain": [1024, 512, 512], "fluid_fraction": fluid, "storage": a.storage,
            "steps": a.steps, "tiles_total": 8192, **out}
    if "static" in out:
        line["speedup_progressive_vs_static"] = round(out["static"]["total_ms"] / out["progressive"]["total_ms"], 3)
    print(json.dumps(line), flush=True)


def c1(a):
    """BASELINE configs[0], the reference's own CPU scenario, end to end on both
    engines in the same run: 500 steps of the 64^3 single-component inflow on
    16^3 tiles (S = 1e-12), the GPU engine (device time, speculative queue)
    against the reference on every host core (wall time), same creation log."""
    import os as _os
    cores = _os.cpu_count() or 1
    sc = S.config1(threshold=1e-12)
    sc.devices = cores  # the reference's workers own tiles by owner % W (engine.cpp:217)
    eng = capi.gpu_engine(sc, storage=a.storage)
    ms, cells, _ = timed(eng, a.steps, chunk=a.steps)
    gpu_log, gpu_c = eng.creation_log(), eng.counters()
    eng.close()
    ref = capi.ref_engine(sc, workers=cores)
    t0 = time.perf_counter()
    ref.step(a.steps)
    ref_s = time.perf_counter() - t0
    same = ref.creation_log() == gpu_log and all(
        ref.counters()[k] == gpu_c[k] for k in ("iteration", "cell_updates", "tiles", "suppressed_expansions"))
    print(json.dumps({"sweep": "c1", "steps": a.steps, "tiles_final": gpu_c["tiles"],
                      "cell_updates": gpu_c["cell_updates"],
                      "gpu_ms": round(ms, 2), "gpu_mlups": round(cells / (ms / 1e3) / 1e6, 1),
                      "ref_s": round(ref_s, 3), "ref_cores": cores,
                      "ref_mlups": round(gpu_c["cell_updates"] / ref_s / 1e6, 2),
                      "speedup": round(ref_s * 1e3 / ms, 1), "same_log_and_counters": same}), flush=True)


def ranks(a):
    from paper_1510_03560_b200 import dist
    for world in (1, 2, 4):
        sc = S.bench_c2()
        sc.devices = max(sc.devices, world)
        engs = [capi.gpu_engine(sc, rank=r, world=world) for r in range(world)]
        if world > 1:
            pools = [e.pool_pointers() for e in engs]
            for r, e in enumerate(engs):
                for q in range(world):
                    if q != r:
                        e.set_peer_pools(q, pools[q])
            for e in engs:
                e.prepare()
        step = (lambda n: engs[0].step(n)) if world == 1 else (lambda n: dist.step_ranks_threaded(engs, n))
        step(100 + a.warmup)
        for e in engs:
            e.sync()
        c0 = engs[0].counters()["cell_updates"]
        t0 = time.perf_counter()
        step(a.steps)
        for e in engs:
            e.sync()
        dt = time.perf_counter() - t0
        cells = engs[0].counters()["cell_updates"] - c0
        print(json.dumps({"sweep": "ranks", "world": world, "gpus": 1, "steps": a.steps,
                          "tiles": engs[0].counters()["tiles"],
                          "tiles_per_rank": [len([t for t in engs[0].tiles() if engs[0].tile_rank(t[0]) == r])
                                             for r in range(world)],
                          "ms_per_step": round(1e3 * dt / a.steps, 3),
                          "mlups_per_comp": round(cells * sc.n_components / dt / 1e6, 1)}), flush=True)
        for e in engs:
            e.close()


def placement(a):
    import numpy as np
    n_dev = 8
    island = np.array([[1 if i // 4 == j // 4 else 0 for j in range(n_dev)] for i in range(n_dev)], np.uint8)
    for policy, name in ((S.POLICY_SIMPLE, "simple"), (S.POLICY_OPTIMIZED, "optimized")):
        sc = S.mpmc_channel(nx=a.n * 2, ny=a.n, nz=a.n, extent=32, threshold=1e-9, devices=n_dev)
        sc.p2p = island
        sc.policy = policy
        eng = capi.gpu_engine(sc)
        ms, cells, _ = timed(eng, a.steps, chunk=a.steps)
        c = eng.counters()
        tiles = eng.tiles()
        owner = {tuple(t[0]): t[1] for t in tiles}
        faces = {"intra": 0, "p2p": 0, "staged": 0}
        for xyz, o in owner.items():
            for ax in range(3):
                for sgn in (-1, 1):
                    nb = list(xyz)
                    nb[ax] += sgn
                    q = owner.get(tuple(nb))
                    if q is None:
                        continue
                    faces["intra" if q == o else ("p2p" if island[o][q] else "staged")] += 1
        E, C = sc.tile_extent, sc.n_components
        per_face = 11 * E * E * C * 8
        print(json.dumps({
            "sweep": "placement", "policy": name, "domain": list(sc.domain), "devices": n_dev,
            "topology": "2 islands x 4 (p2p inside, staged across)", "steps": a.steps,
            "tiles": c["tiles"], "tiles_per_device": [sum(1 for o in owner.values() if o == d) for d in range(n_dev)],
            "modeled_bytes": {"intra": c["bytes"][0], "p2p": c["bytes"][1], "staged": c["bytes"][2]},
            "final_mesh_face_links": faces,
            "cross_device_bytes_per_step": {"p2p": faces["p2p"] * per_face, "staged": faces["staged"] * per_face},
            "gpu_ms": round(ms, 1)}), flush=True)
        eng.close()


def main():
    p = argparse.ArgumentParser()
    p.add_argument("what", choices=["c1", "c5", "c3", "c4", "placement", "ranks"])
    p.add_argument("--n", type=int, default=None)
    p.add_argument("--steps", type=int, default=None)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--every", type=int, default=25)
    p.add_argument("--storage", choices=["ab", "aa"], default="ab",
                   help="population storage: two buffers (ab) or one in-place A-A buffer (aa)")
    p.add_argument("--static", action="store_true", help="c4: also the static full mesh")
    p.add_argument("--variant", type=int, default=0, help="c4: fused-kernel variant / modifiers (plbm_gpu.h)")
    p.add_argument("--extents", type=int, nargs="+", default=[16, 32, 64], help="c5: tile extents")
    p.add_argument("--comps", type=int, nargs="+", default=[1, 2, 3], help="c5: component counts")
    a = p.parse_args()
    if a.what == "c5":
        a.n = a.n or 256
        a.steps = a.steps or 20
        c5(a)
    elif a.what == "c1":
        a.steps = a.steps or 500
        c1(a)
    elif a.what == "c4":
        a.steps = a.steps or 400
        a.every = 50
        c4(a)
    elif a.what == "ranks":
        a.steps = a.steps or 30
        ranks(a)
    elif a.what == "placement":
        a.n = a.n or 512
        a.steps = a.steps or 400
        placement(a)
    else:
        a.n = a.n or 512
        a.steps = a.steps or 300
        c3(a)


if __name__ == "__main__":
    main()
