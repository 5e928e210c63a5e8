#!/usr/bin/env python
"""Benchmark: MLUPS per component of the progressive-mesh MPMC D3Q19 step loop.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload (BASELINE.json configs[1]): D3Q19 two-component MPMC
(Peng-Robinson liquid/vapour + ideal-like light gas, g_cross = 0.08) released
from a ramped liquid sphere into a 256^3 domain, progressive mesh of 32^3
subdomains, S = 1e-9, FP64.  The mesh is grown for --pre-steps steps before
the W warm-up steps so the timed steps run on the developed mesh (the state at
that point is the benchmark's input).  Each step reads+writes ~10 GB, far more
than the 126 MB L2, so no explicit flush is needed between steps.

One JSON line on rank 0.  `value` is device-timed (CUDA events on the engine's
stream, max over ranks); `e2e` is the same metric through the C-ABI with the
per-step host read of the report counters, host-clock timed; `roofline` is the
fused kernel's algorithmic bytes (304 B per cell update per component, SURVEY
§8(d)) over its CUDA-event duration; `cpu_baseline` is the reference itself
(oracle/_ref, built from the reference sources) on the host cores.

--impl reference times the reference CPU implementation (oracle/_ref) on the
box's host cores on a bounded 128^3 sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

from paper_1510_03560_b200 import scenario as S  # noqa: E402

BYTES_PER_CELL_COMP = 2 * 19 * 8  # f read + f write, FP64
FALLBACK_HBM_GBS = 6650.0         # /opt/skills/guides/B200_PROFILING.md


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=30)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--config", choices=["c2", "c2_static", "c1"], default="c2")
    p.add_argument("--pre-steps", type=int, default=100)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--cpu-seconds", type=float, default=15.0)
    p.add_argument("--variant", type=int, default=0, help="fused-kernel variant (plbm_gpu.h)")
    p.add_argument("--dist-backend", default="nccl", help="nccl (one GPU per rank) or gloo (tests)")
    return p.parse_args()


def workload(cfg: str, world: int = 1):
    if cfg == "c2" and world > 1:
        return S.mpmc_release_weak(world), \
            f"C2 weak-scaled: {world} x (256^3 2-comp MPMC sphere release) along x, 32^3 subdomains, progressive S=1e-9, owners sharded over {world} GPUs"
    if cfg == "c2":
        return S.mpmc_release(n=256, extent=32, threshold=1e-9), \
            "C2: D3Q19 2-comp MPMC (PR liquid/vapour + ideal-like) sphere release, 256^3, 32^3 subdomains, progressive S=1e-9"
    if cfg == "c2_static":
        return S.mpmc_release(n=256, extent=32, mode=S.MODE_STATIC), \
            "C2-static: D3Q19 2-comp MPMC sphere release, 256^3 full static mesh, 32^3 subdomains"
    return S.config1(threshold=1e-12), \
        "C1: D3Q19 1-comp ideal gas, moving box inflow into 64^3, 16^3 subdomains, progressive S=1e-12"


def cpu_sample_scenario():
    """Bounded CPU sample: same physics / tile size / components at 128^3,
    static mesh (every tile active = the developed-mesh per-cell cost)."""
    return S.mpmc_release(n=128, extent=32, mode=S.MODE_STATIC)


def hbm_peak():
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback"


def run_reference_cpu(seconds: float, warmup: int = 1, max_steps: int = 10**9):
    """Times the reference (oracle/_ref/libplbm_ref.so, compiled from the
    reference sources) on the host cores: MLUPS per component."""
    from paper_1510_03560_b200 import capi
    cores = os.cpu_count() or 1
    sc = cpu_sample_scenario()
    sc.devices = cores  # tiles go to worker owner % W (engine.cpp:217)
    eng = capi.ref_engine(sc, workers=cores)
    eng.step(warmup)
    c0 = eng.counters()["cell_updates"]
    t0 = time.perf_counter()
    n = 0
    while n < max_steps:
        eng.step(1)
        n += 1
        if time.perf_counter() - t0 > seconds:
            break
    dt = time.perf_counter() - t0
    cells = eng.counters()["cell_updates"] - c0
    eng.close()
    value = cells * sc.n_components / dt / 1e6
    sample = f"reference (oracle/_ref) 128^3 2-comp MPMC static, 32^3 tiles, {n} steps after {warmup} warm-up, {cores} worker threads"
    return value, cores, sample, n, dt


class ClockSampler:
    def __init__(self, path, index=0):
        self.path, self.index, self.proc = path, index, None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=self.fh, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            self.proc.wait()
            self.fh.close()

    def summary(self):
        try:
            rows = [r.split(",") for r in open(self.path).read().strip().splitlines()]
        except Exception:
            return None
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            if len(r) < 8:
                continue
            try:
                sm.append(float(r[0]))
                mx = float(r[1])
            except ValueError:
                continue
            for k, nm in enumerate(names):
                if r[4 + k].strip().lower() == "active":
                    reasons.add(nm)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def main():
    a = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if a.impl == "reference":
        if rank != 0:
            return
        value, cores, sample, n, dt = run_reference_cpu(a.cpu_seconds, warmup=a.warmup,
                                                        max_steps=max(a.steps, 1))
        _, name = workload(a.config)
        line = {"metric": "MLUPS per component (D3Q19 MPMC)", "value": round(value, 3),
                "unit": "MLUPS/comp", "impl": "reference", "n_gpus": a.gpus, "steps": n,
                "warmup": a.warmup, "ms_per_step": round(1000 * dt / max(n, 1), 3),
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic", "config": {"workload": name, "sample": sample},
                "cpu_baseline": {"value": round(value, 3), "unit": "MLUPS/comp", "cores": cores,
                                 "kind": "reference", "sample": sample},
                "e2e": {"value": round(value, 3), "unit": "MLUPS/comp", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return

    import torch
    ndev = torch.cuda.device_count()
    gpu = local % max(ndev, 1)
    torch.cuda.set_device(gpu)
    dist = None
    if world > 1:
        import torch.distributed as dist
        if a.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", gpu))
        else:
            dist.init_process_group(a.dist_backend)
    from paper_1510_03560_b200 import capi
    from paper_1510_03560_b200.dist import DistStepper
    sc, name = workload(a.config, world)
    C = sc.n_components
    eng = capi.gpu_engine(sc, device=gpu, rank=rank, world=world)
    eng.set_kernel_variant(a.variant)
    stream = torch.cuda.ExternalStream(eng.stream(), device=torch.device("cuda", gpu))
    if world > 1:
        stepper = DistStepper(eng, dist, gpu)
        run = stepper.step
    else:
        run = eng.step

    run(a.pre_steps)
    run(a.warmup)
    tiles_at_start = eng.counters()["tiles"]

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    os.makedirs(os.path.join(REPO, "gpurun_out"), exist_ok=True)
    # ---- device-timed region -------------------------------------------------
    # (no per-kernel events inside it: they cost ~3 %; the kernel split for
    # the roofline comes from a separate profiled pass of the same steps below)
    eng.reset_kernel_stats()
    c0 = eng.counters()["cell_updates"]
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(os.path.join(REPO, "gpurun_out", f"clocks_r{rank}.csv"), local) as clk:
        barrier()
        ev0.record(stream)
        run(a.steps)
        ev1.record(stream)
        barrier()
    ms = ev0.elapsed_time(ev1)
    cells = eng.counters()["cell_updates"] - c0
    launches = eng.kernel_stats()["kernels_launched"]
    tiles_at_end = eng.counters()["tiles"]

    # ---- per-kernel CUDA events (roofline of the fused kernel) ----------------
    eng.reset_kernel_stats()
    eng.set_profiling(True)
    run(a.steps)
    barrier()
    ks = eng.kernel_stats()
    eng.set_profiling(False)

    # ---- end to end through the C-ABI: step + per-step host read of the
    # report counters (what the reference driver reads each step) -------------
    eng.reset_kernel_stats()
    e0 = eng.counters()["cell_updates"]
    barrier()
    t0 = time.perf_counter()
    for _ in range(a.steps):
        run(1)
        eng.counters()
    barrier()
    e_dt = time.perf_counter() - t0
    e_cells = eng.counters()["cell_updates"] - e0
    e_ks = eng.kernel_stats()

    # ---- max over ranks / sums -------------------------------------------------
    # cell_updates is a global count (every rank's mirror sees all tiles), so
    # the job total is taken once; times are the max over ranks.
    tdev = "cuda" if (dist is None or a.dist_backend == "nccl") else "cpu"
    t = torch.tensor([ms, e_dt], dtype=torch.float64, device=tdev)
    if dist is not None:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max, e_dt_max = float(t[0]), float(t[1])
    xb = torch.tensor([float(eng.exchange_bytes()["bytes_per_step"])], dtype=torch.float64, device=tdev)
    if dist is not None:
        dist.all_reduce(xb)  # job total per step
    nvlink_bytes = int(xb[0])
    cells_all, e_cells_all = float(cells), float(e_cells)
    if rank != 0:
        if dist is not None:
            dist.destroy_process_group()
        return

    value = cells_all * C / (ms_max / 1e3) / 1e6
    e2e = e_cells_all * C / e_dt_max / 1e6
    peak, peak_kind = hbm_peak()
    achieved = (ks["main_cell_updates"] * C * BYTES_PER_CELL_COMP / (ks["main_ms"] / 1e3) / 1e9
                if ks["main_ms"] > 0 else None)
    # DRAM traffic of the fused kernel from the committed ncu --set full capture
    # (profiles/ncu_kmain_summary.json), per cell update per component, scaled
    # to this run's average launch.
    traffic = None
    prof = os.path.join(REPO, "profiles", "ncu_kmain_summary.json")
    if os.path.exists(prof) and ks["main_launches"]:
        try:
            bpc = json.load(open(prof))["dram_bytes_per_cell_comp"]
            traffic = round(bpc * ks["main_cell_updates"] / ks["main_launches"] * C)
        except Exception:
            traffic = None
    line = {
        "metric": "MLUPS per component (D3Q19 MPMC)",
        "value": round(value, 2), "unit": "MLUPS/comp", "n_gpus": world, "steps": a.steps,
        "warmup": a.warmup, "ms_per_step": round(ms_max / a.steps, 4), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": name, "pre_steps": a.pre_steps, "tiles": [tiles_at_start, tiles_at_end],
                   "components": C, "tile_extent": sc.tile_extent,
                   "parallelism": f"tile-sharded x{world} (owner % world), NVLink peer loads" if world > 1 else "1 GPU",
                   "l2": "per-step working set ~10 GB >> 126 MB L2 (no flush needed)",
                   "mlups_cells": round(value / C, 2)},
        "e2e": {"value": round(e2e, 2), "unit": "MLUPS/comp",
                "h2d_bytes_per_step": int(e_ks["h2d_bytes"] / max(a.steps, 1)),
                "d2h_bytes_per_step": int(e_ks["d2h_bytes"] / max(a.steps, 1))},
        "gpu_launches": int(launches),
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1) if achieved else None,
                     "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4) if achieved else None,
                     "traffic": traffic, "peak_kind": peak_kind,
                     "algorithmic_bytes_per_launch": round(BYTES_PER_CELL_COMP * C * ks["main_cell_updates"] / max(ks["main_launches"], 1)),
                     "kernel": "k_main (fused pull-stream + psi + forces + BGK collide)",
                     "kernel_ms_avg": round(ks["main_ms"] / max(ks["main_launches"], 1), 4),
                     "face_ms_avg": round(ks["face_ms"] / max(ks["face_launches"], 1), 4)},
        "clocks": clk.summary(),
    }
    if world > 1:
        # real cross-GPU volume per step (routing tables) next to the
        # reference's modeled classes (record_exchange), SURVEY §8(f)4
        c = eng.counters()
        line["exchange"] = {"nvlink_read_bytes_per_step": nvlink_bytes,
                            "nvlink_GBs": round(nvlink_bytes / (ms_max / a.steps / 1e3) / 1e9, 1),
                            "modeled_bytes_total": {"intra": c["bytes"][0], "p2p": c["bytes"][1],
                                                    "staged": c["bytes"][2]}}
    if not a.no_cpu_baseline and world == 1:
        try:
            v, cores, sample, _, _ = run_reference_cpu(a.cpu_seconds)
            line["cpu_baseline"] = {"value": round(v, 3), "unit": "MLUPS/comp", "cores": cores,
                                    "kind": "reference", "sample": sample}
        except Exception as ex:  # the reference shim is built here and travels
            line["cpu_baseline"] = {"value": None, "unit": "MLUPS/comp", "cores": os.cpu_count(),
                                    "kind": "reference", "sample": f"unavailable: {ex}"}
    print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
