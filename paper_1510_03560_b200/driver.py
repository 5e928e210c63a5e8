"""The reference's simulation driver on the B200 engine.

`run_scenario` mirrors engine::run_scenario (proj/src/engine.cpp:580-704): it
steps the engine, keeps the reporting windows, takes snapshots and writes the
same three report files with the same formats (proj/src/report.cpp:24-81):

    <out>/time_series.csv   one row per report interval (and the last step)
    <out>/creation_log.csv  TileMap::creation_log()
    <out>/summary.json      RunSummary as nlohmann::json::dump(2)
    <out>/snapshots/<field>_c<k>_i<iter>.raw/.meta[/.pgm]  (dump.cpp:59-125)

Counters, creation log, byte classes and snapshot files are identical to the
reference's for the same scenario (tests/test_output_path.py); the timing
columns are this engine's own wall-clock.  `workers` is reported as the
reference would (one per device) — there are no CPU worker threads here.
"""
from __future__ import annotations

import json
import os
import time
from typing import Iterable, Optional

from . import capi
from . import scenario as S

# proj/src/tile.cpp:15-19
FOOTPRINT_FORMULA = ("gcells*(n_comp*(2*q+8)*8 + 1), gcells=(extent+2)^2*(extent+2 if "
                     "3-D else 1); doubles: 2 population buffers (q each), rho, "
                     "ux/uy/uz, prev ux/uy/uz, psi; plus 1 byte solid mask")


def _g17(v: float) -> str:
    """std::ostream with precision(17): %.17g."""
    return "%.17g" % v


def _mlups(updates: int, seconds: float) -> float:  # proj/src/report.cpp:10-13
    return 0.0 if seconds <= 0.0 else updates / seconds / 1e6


def run_scenario(sc: S.Scenario, output_dir: str, iterations: int, report_interval: int = 10,
                 snapshot_interval: int = 0, snapshot_fields: Iterable[str] = ("rho",),
                 snapshot_pgm: bool = False, name: str = "scenario", workers: int = 0,
                 device: int = 0, engine: Optional[capi.GpuEngine] = None) -> dict:
    fields = list(snapshot_fields)
    os.makedirs(output_dir, exist_ok=True)
    snapshots = snapshot_interval > 0
    if snapshots:
        os.makedirs(os.path.join(output_dir, "snapshots"), exist_ok=True)
    eng = engine or capi.gpu_engine(sc, device=device, capture=snapshots and "psi" in fields)
    C = sc.n_components
    res = {"rows": [], "snapshot_bases": [], "aborted": False, "abort_context": ""}

    def take_snapshot(it: int) -> None:
        for f in fields:
            for c in range(C):
                base = "%s_c%d_i%07d" % (f, c, it)
                eng.dump_field(f, c, it, os.path.join(output_dir, "snapshots", base), snapshot_pgm)
                res["snapshot_bases"].append("snapshots/" + base)

    if snapshots:
        take_snapshot(0)
    bbox = sc.domain[0] * sc.domain[1] * sc.domain[2]
    cnt = eng.counters()
    peak = cnt["bytes_resident"]
    total_s = win_s = 0.0
    win_upd = win_steps = 0
    last = {"negative_populations": 0, "psi_clamps": 0, "suppressed_expansions": 0}

    def flush_row(it: int) -> None:
        nonlocal win_s, win_upd, win_steps
        c = eng.counters()
        row = {"iteration": it, "tiles": c["tiles"], "active_cells": c["active_cells"],
               "bytes": list(c["bytes"]), "window_seconds": win_s,
               "window_mlups": _mlups(win_upd, win_s),
               "window_mlups_bbox": _mlups(win_steps * bbox, win_s)}
        for k in last:
            row["window_" + k] = c[k] - last[k]
            last[k] = c[k]
        res["rows"].append(row)
        win_s, win_upd, win_steps = 0.0, 0, 0

    for k in range(1, iterations + 1):
        before = eng.counters()["cell_updates"]
        t0 = time.perf_counter()
        try:
            eng.step(1)
        except S.EngineError as e:
            res["aborted"], res["abort_context"] = True, str(e)
            break
        dt = time.perf_counter() - t0
        c = eng.counters()
        total_s += dt
        win_s += dt
        win_upd += c["cell_updates"] - before
        win_steps += 1
        peak = max(peak, c["bytes_resident"])
        if k % report_interval == 0 or k == iterations:
            flush_row(k)
        if snapshots and (k % snapshot_interval == 0 or k == iterations):
            take_snapshot(k)
    c = eng.counters()
    if res["aborted"] and win_steps > 0:
        flush_row(c["iteration"])

    owners = [o for _, o, _ in eng.tiles()]
    per_dev = [owners.count(d) for d in range(sc.devices)]
    summary = {
        "name": name,
        "mode": "static" if sc.mode == S.MODE_STATIC else "progressive",
        "policy": "simple" if sc.policy == S.POLICY_SIMPLE else "optimized",
        "stencil": "D3Q19",
        "devices": sc.devices,
        "workers": workers if workers > 0 else sc.devices,
        "tile_extent": sc.tile_extent,
        "domain": list(sc.domain),
        "iterations": c["iteration"],
        "total_cell_updates": c["cell_updates"],
        "compute_seconds": total_s,
        "mlups": _mlups(c["cell_updates"], total_s),
        "mlups_bbox": _mlups(c["iteration"] * bbox, total_s),
        "peak_resident_bytes": peak,
        "footprint_formula": FOOTPRINT_FORMULA,
        "tiles_final": c["tiles"],
        "active_cells_final": c["active_cells"],
        "bytes": {"intra": c["bytes"][0], "p2p": c["bytes"][1], "staged": c["bytes"][2]},
        "diagnostics": {"negative_populations": c["negative_populations"],
                        "psi_clamps": c["psi_clamps"],
                        "suppressed_expansions": c["suppressed_expansions"],
                        "zero_rho_forcings": c["zero_rho_forcings"]},
        "per_device_tiles": per_dev,
        "status": ("aborted: " + res["abort_context"]) if res["aborted"] else "completed",
    }
    _write_time_series(res["rows"], os.path.join(output_dir, "time_series.csv"))
    _write_creation_log(eng.creation_log(), os.path.join(output_dir, "creation_log.csv"))
    _write_summary(summary, os.path.join(output_dir, "summary.json"))
    res["summary"] = summary
    if engine is None:
        eng.close()
    return res


def _write_time_series(rows, path: str) -> None:  # proj/src/report.cpp:24-39
    with open(path, "w") as fh:
        fh.write("iteration,tiles,active_cells,bytes_intra,bytes_p2p,bytes_staged,"
                 "window_seconds,window_mlups,window_mlups_bbox,"
                 "window_negative_populations,window_psi_clamps,"
                 "window_suppressed_expansions\n")
        for r in rows:
            fh.write(",".join([str(r["iteration"]), str(r["tiles"]), str(r["active_cells"]),
                               *map(str, r["bytes"]), _g17(r["window_seconds"]),
                               _g17(r["window_mlups"]), _g17(r["window_mlups_bbox"]),
                               str(r["window_negative_populations"]), str(r["window_psi_clamps"]),
                               str(r["window_suppressed_expansions"])]) + "\n")


def _write_creation_log(log, path: str) -> None:  # proj/src/report.cpp:41-49
    with open(path, "w") as fh:  # trigger: "init" or the face name ("-x" .. "+z")
        fh.write("iteration,tile_x,tile_y,tile_z,trigger_face,owner_device\n")
        for it, (x, y, z), trig, owner in log:
            fh.write(f"{it},{x},{y},{z},{trig},{owner}\n")


def _write_summary(s: dict, path: str) -> None:  # proj/src/report.cpp:51-79
    # nlohmann::json objects are std::map-ordered (sorted keys), dump(2)
    with open(path, "w") as fh:
        fh.write(json.dumps(s, indent=2, sort_keys=True) + "\n")
