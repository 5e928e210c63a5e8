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
stream, max over ranks); `e2e` is the same metric through the C-ABI in the
reference driver's loop (one step call + the report counters per iteration,
then the final rho snapshot gathered to host memory), host-clock timed; `roofline` is the
fused kernel's algorithmic bytes (304 B per cell update per component, SURVEY
§8(d)) over its CUDA-event duration; `cpu_baseline` is the reference itself
(oracle/_ref, built from the reference sources) on the host cores.

--impl reference times the reference CPU implementation (oracle/_ref, built
from the reference sources) on the box's host cores on the SAME workload:
the same pre-steps grow the mesh, the same warm-up, then the timed steps (the
config dict is identical in both lines).  Configs whose reference footprint
exceeds the host's memory (C3/C4/C5 at 512^3+) fall back to a bounded static
sample of the same physics and say so.
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
    p.add_argument("--steps", type=int, default=100)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--config", choices=["c2", "c2_static", "c1", "c3", "c3_static", "c4", "c5"], default="c2")
    p.add_argument("--pre-steps", type=int, default=None,
                   help="steps before warm-up that grow the mesh (default per config)")
    p.add_argument("--extent", type=int, default=32, help="c5: subdomain size E")
    p.add_argument("--components", type=int, default=2, help="c5: component count C")
    p.add_argument("--snapshot-every", type=int, default=0,
                   help="e2e loop: gather the rho field of every component to host memory every N "
                        "steps (the driver's snapshot_interval; default 0 = the reference's default)")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--cpu-seconds", type=float, default=20.0)
    p.add_argument("--variant", type=int, default=0, help="fused-kernel variant (plbm_gpu.h)")
    p.add_argument("--storage", choices=["ab", "aa"], default="ab",
                   help="population storage: A-B double buffer or A-A in place (one buffer)")
    p.add_argument("--dist-backend", default="nccl", help="nccl (one GPU per rank) or gloo (tests)")
    return p.parse_args()


# name -> (builder(world, args), description, default pre-steps, scaling at N > 1)
def workload(a, world: int = 1):
    cfg = a.config
    if cfg == "c2" and world > 1:
        sc = S.mpmc_release_weak(world)
        return sc, (f"C2 weak-scaled: {world} x (256^3 2-comp MPMC sphere release) along x, 32^3 "
                    f"subdomains, progressive S=1e-9"), 100, "weak"
    if cfg == "c2":
        return S.bench_c2(), ("C2: D3Q19 2-comp MPMC (PR liquid/vapour + ideal-like) sphere release, "
                              "256^3, 32^3 subdomains, progressive S=1e-9"), 100, "weak"
    if cfg == "c2_static":
        return S.bench_c2(S.MODE_STATIC), "C2-static: 256^3 2-comp MPMC sphere release, full static mesh, 32^3 subdomains", 0, "weak"
    if cfg == "c3":
        sc = S.mpmc_release(n=512, extent=32, threshold=1e-9, devices=S.BENCH_DEVICES)
        return sc, "C3 progressive: 512^3 2-comp MPMC sphere release, 32^3 subdomains, S=1e-9", 100, "strong"
    if cfg == "c3_static":
        sc = S.mpmc_release(n=512, extent=32, mode=S.MODE_STATIC, devices=S.BENCH_DEVICES)
        return sc, "C3 static: 512^3 2-comp MPMC sphere release, full static mesh (4096 tiles), 32^3 subdomains", 0, "strong"
    if cfg == "c4":
        sc = S.mpmc_channel(devices=S.BENCH_DEVICES)
        return sc, ("C4: 1024x512x512 3-D channel network (LBMGEO generator, seed 1510), 2-comp MPMC "
                    "liquid sphere in the inlet channel, 32^3 subdomains, progressive S=1e-9"), 400, "strong"
    if cfg == "c5":
        sc = S.mpmc_release(n=512, extent=a.extent, mode=S.MODE_STATIC, n_components=a.components,
                            devices=S.BENCH_DEVICES)
        return sc, (f"C5: 512^3 static MPMC sphere release, {a.extent}^3 subdomains, "
                    f"{a.components} component(s)"), 0, "strong"
    return S.config1(threshold=1e-12), ("C1: D3Q19 1-comp ideal gas, moving box inflow into 64^3, "
                                        "16^3 subdomains, progressive S=1e-12"), 0, "weak"


def bench_config(a, sc, name, pre):
    """The workload identity (identical in both arms' JSON lines)."""
    return {"workload": name, "domain": list(sc.domain), "tile_extent": sc.tile_extent,
            "components": sc.n_components, "mode": "static" if sc.mode == S.MODE_STATIC else "progressive",
            "threshold": sc.threshold, "pre_steps": pre, "simulated_devices": sc.devices,
            "l2": "per-step working set >= 0.6 GB >> 126 MB L2 at every config (no flush needed)",
            "storage": getattr(a, "storage", "ab")}


def hbm_peak():
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback"


def reference_threads(sc) -> int:
    """Worker threads the reference engine can use on this host: tiles go to
    worker owner % W (engine.cpp:214-218), so W <= simulated devices."""
    return max(1, min(os.cpu_count() or 1, sc.devices))


def fits_host(sc) -> bool:
    """The reference keeps every tile with a ghost ring and two population
    buffers on the host (tile.cpp:7-13): 28.97 MB per 32^3 2-comp tile."""
    g = (sc.tile_extent + 2) ** 3
    per_tile = g * (sc.n_components * (2 * 19 + 8) * 8 + 1)
    tiles = 1
    for d in sc.domain:
        tiles *= d // sc.tile_extent
    try:
        avail = os.sysconf("SC_AVPHYS_PAGES") * os.sysconf("SC_PAGE_SIZE")
    except (ValueError, OSError):
        avail = 0
    return per_tile * tiles < 0.7 * avail


def run_reference_arm(a, sc, pre, steps, warmup):
    """The reference's own CPU engine (oracle/_ref/libplbm_ref.so, compiled
    from /root/reference/proj/src) through make_state + Engine::step on the
    SAME workload: pre-steps grow the mesh, `warmup` untimed steps, then
    `steps` timed steps, each a whole Engine::step over every active tile.
    Returns (MLUPS/comp, threads, sample description, steps, seconds)."""
    from paper_1510_03560_b200 import capi
    W = reference_threads(sc)
    eng = capi.ref_engine(sc, workers=W)
    eng.step(pre + warmup)
    c0 = eng.counters()["cell_updates"]
    t0 = time.perf_counter()
    eng.step(steps)
    dt = time.perf_counter() - t0
    cells = eng.counters()["cell_updates"] - c0
    tiles = eng.counters()["tiles"]
    eng.close()
    sample = (f"reference (oracle/_ref, built from the reference sources) on the same workload: "
              f"{pre} pre-steps + {warmup} warm-up, then {steps} timed steps on {tiles} tiles, {W} worker threads")
    return cells * sc.n_components / dt / 1e6, W, sample, steps, dt


def run_cpu_sample(sc_full, seconds: float):
    """Bounded cpu_baseline sample (about `seconds` of CPU work): the same
    physics, tile size and component count on the full static mesh of the
    workload's domain (= the developed progressive mesh's per-cell cost) when
    the reference's host footprint fits, else a 256^3 static block of it."""
    from paper_1510_03560_b200 import capi
    import copy
    sc = copy.deepcopy(sc_full)
    sc.mode = S.MODE_STATIC
    if not fits_host(sc):
        sc = S.mpmc_release(n=256, extent=sc_full.tile_extent, mode=S.MODE_STATIC,
                            n_components=sc_full.n_components, devices=sc_full.devices)
    W = reference_threads(sc)
    eng = capi.ref_engine(sc, workers=W)
    eng.step(1)
    c0 = eng.counters()["cell_updates"]
    t0 = time.perf_counter()
    n = 0
    while True:
        eng.step(1)
        n += 1
        if time.perf_counter() - t0 > seconds:
            break
    dt = time.perf_counter() - t0
    cells = eng.counters()["cell_updates"] - c0
    eng.close()
    sample = (f"reference (oracle/_ref) static {sc.domain[0]}x{sc.domain[1]}x{sc.domain[2]}, "
              f"{sc.tile_extent}^3 tiles, {sc.n_components} comp, {n} steps after 1 warm-up, {W} worker threads")
    return cells * sc.n_components / dt / 1e6, W, sample


def nvlink_bytes(index: int):
    """NVLink data bytes this GPU sent / received so far (NVML field values
    NVLINK_THROUGHPUT_DATA_TX / _RX, KiB counters summed over the links), or
    None where NVML does not expose them."""
    try:
        import pynvml
        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(index)
        vals = pynvml.nvmlDeviceGetFieldValues(h, [pynvml.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX,
                                                   pynvml.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_RX])
        if any(v.nvmlReturn != 0 for v in vals):
            return None
        return int(vals[0].value.ullVal) * 1024, int(vals[1].value.ullVal) * 1024
    except Exception:
        return None


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
    sc, name, pre_default, scaling = workload(a, world)
    pre = pre_default if a.pre_steps is None else a.pre_steps
    config = bench_config(a, sc, name, pre)

    if a.impl == "reference":
        if rank != 0:
            return
        ref_sc = sc
        if world > 1 and a.config == "c2":
            ref_sc = S.bench_c2()  # the per-GPU block: same per-cell work, 1/N of the job
        if not fits_host(ref_sc):
            value, cores, sample = run_cpu_sample(ref_sc, a.cpu_seconds)
            n, dt = 0, 0.0
        else:
            value, cores, sample, n, dt = run_reference_arm(a, ref_sc, pre, max(a.steps, 1), a.warmup)
        if ref_sc is not sc:
            sample += f" (one 256^3 block of the {world}-block weak-scaled job: the per-cell work is identical)"
        line = {"metric": "MLUPS per component (D3Q19 MPMC)", "value": round(value, 3),
                "unit": "MLUPS/comp", "impl": "reference", "n_gpus": a.gpus, "steps": n or a.steps,
                "warmup": a.warmup, "ms_per_step": round(1000 * dt / max(n, 1), 3),
                "higher_is_better": True, "scaling": scaling, "vs_baseline": None, "dtype": "f64",
                "data": "synthetic", "config": config,
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
    C = sc.n_components
    eng = capi.gpu_engine(sc, device=gpu, rank=rank, world=world, storage=a.storage)
    eng.set_kernel_variant(a.variant)
    stream = torch.cuda.ExternalStream(eng.stream(), device=torch.device("cuda", gpu))
    if world > 1:
        stepper = DistStepper(eng, dist, gpu)
        run = stepper.step
    else:
        run = eng.step

    run(pre)
    run(a.warmup)

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    # ---- end to end through the C-ABI, the reference driver's loop, on the
    # same steps the reference arm times (right after pre-steps + warm-up)
    # (engine::run_scenario, proj/src/engine.cpp:640-668): one plbm_gpu_step
    # per iteration, the report counters read after every step (a superset of
    # flush_row's reads at report_interval), and with --snapshot-every N the
    # rho field of every component gathered into a host grid every N steps
    # (take_snapshot; the reference's default snapshot_interval is 0) -------
    eng.reset_kernel_stats()
    e0 = eng.counters()["cell_updates"]
    barrier()
    t0 = time.perf_counter()
    for k in range(1, a.steps + 1):
        run(1)
        eng.counters()
        if world == 1 and a.snapshot_every and k % a.snapshot_every == 0:
            for c in range(C):
                eng.gather_field("rho", c)  # host grid (counted in d2h_bytes)
    barrier()
    e_dt = time.perf_counter() - t0
    e_cells = eng.counters()["cell_updates"] - e0
    e_ks = eng.kernel_stats()

    os.makedirs(os.path.join(REPO, "gpurun_out"), exist_ok=True)
    # ---- device-timed region -------------------------------------------------
    # (no per-kernel events inside it: they cost ~3 %; the kernel split for
    # the roofline comes from a separate profiled pass of the same steps below)
    eng.reset_kernel_stats()
    c0 = eng.counters()["cell_updates"]
    tiles_at_start = eng.counters()["tiles"]
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(os.path.join(REPO, "gpurun_out", f"clocks_r{rank}.csv"), local) as clk:
        barrier()
        nvl0 = nvlink_bytes(gpu)
        ev0.record(stream)
        run(a.steps)
        ev1.record(stream)
        barrier()
        nvl1 = nvlink_bytes(gpu)
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

    # ---- max over ranks / sums -------------------------------------------------
    # cell_updates is a global count (every rank's mirror sees all tiles), so
    # the job total is taken once; times are the max over ranks.
    tdev = "cuda" if (dist is None or a.dist_backend == "nccl") else "cpu"
    t = torch.tensor([ms, e_dt], dtype=torch.float64, device=tdev)
    if dist is not None:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max, e_dt_max = float(t[0]), float(t[1])
    # cross-GPU bytes per step: from the routing tables (what the kernels read
    # from peer pools) and measured by NVML (NVLink data TX / RX of the timed
    # steps); job totals over the ranks
    hw = [float(nvl1[0] - nvl0[0]), float(nvl1[1] - nvl0[1])] if nvl0 and nvl1 else [-1.0, -1.0]
    xb = torch.tensor([float(eng.exchange_bytes()["bytes_per_step"])] + hw, dtype=torch.float64, device=tdev)
    if dist is not None:
        dist.all_reduce(xb)  # job totals
    table_bytes = int(xb[0])
    nvml_tx, nvml_rx = float(xb[1]), float(xb[2])
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
    if os.path.exists(prof) and ks["main_launches"] and a.config == "c2":
        try:
            bpc = json.load(open(prof))["dram_bytes_per_cell_comp"]
            traffic = round(bpc * ks["main_cell_updates"] / ks["main_launches"] * C)
        except Exception:
            traffic = None
    line = {
        "metric": "MLUPS per component (D3Q19 MPMC)",
        "value": round(value, 2), "unit": "MLUPS/comp", "n_gpus": world, "steps": a.steps,
        "warmup": a.warmup, "ms_per_step": round(ms_max / a.steps, 4), "higher_is_better": True,
        "scaling": scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config,
        "run": {"tiles": [tiles_at_start, tiles_at_end], "mlups_cells": round(value / C, 2),
                "parallelism": f"tile-sharded x{world} (owner % world), NVLink peer loads" if world > 1 else "1 GPU"},
        "e2e": {"value": round(e2e, 2), "unit": "MLUPS/comp",
                "h2d_bytes_per_step": int(e_ks["h2d_bytes"] / max(a.steps, 1)),
                "d2h_bytes_per_step": int(e_ks["d2h_bytes"] / max(a.steps, 1)),
                "loop": "plbm_gpu_step(h, 1) + plbm_gpu_counters per iteration" +
                        (f", rho snapshot of every component to a host grid every {a.snapshot_every} steps"
                         if a.snapshot_every else " (snapshot_interval 0, the reference driver's default)"),
                "copies": "a step has no host input (the lattice state is resident, as in the reference's "
                          "run loop); its result read each step is the report counters (D2H, counted); "
                          "--snapshot-every N adds the field read-backs the reference's snapshots do"},
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
        hw_ok = nvml_tx >= 0 and nvml_rx >= 0
        line["exchange"] = {"routing_table_bytes_per_step": table_bytes,
                            "routing_table_GBs": round(table_bytes / (ms_max / a.steps / 1e3) / 1e9, 1),
                            "nvml_nvlink_tx_bytes_per_step": round(nvml_tx / a.steps) if hw_ok else None,
                            "nvml_nvlink_rx_bytes_per_step": round(nvml_rx / a.steps) if hw_ok else None,
                            "nvml_nvlink_GBs": (round(nvml_rx / a.steps / (ms_max / a.steps / 1e3) / 1e9, 1)
                                                if hw_ok else None),
                            "modeled_bytes_total": {"intra": c["bytes"][0], "p2p": c["bytes"][1],
                                                    "staged": c["bytes"][2]},
                            "ranks": world, "protocol": "plbm_gpu_step: device rank barriers + replicated expansion"}
    if not a.no_cpu_baseline and world == 1:
        try:
            v, cores, sample = run_cpu_sample(sc, a.cpu_seconds)
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
