"""The reference's simulation driver on the B200 engine.

`run_scenario` mirrors engine::run_scenario (proj/src/engine.cpp:580-704): it
steps the engine, keeps the reporting windows, takes snapshots and writes the
same three report files with the same formats (proj/src/report.cpp:24-81):

    <out>/time_series.csv   one row per report interval (and the last step)
    <out>/creation_log.csv  TileMap::creation_log()
    <out>/summary.json      RunSummary as nlohmann::json::dump(2)
    <out>/snapshots/<field>_c<k>_i<iter>.raw/.meta[/.pgm]  (dump.cpp:59-125)

`run_compare` mirrors the compare mode (proj/src/cli.cpp:133-157): both
modes under <out>/static and <out>/progressive, every snapshot pair diffed,
<out>/compare.csv and <out>/compare_summary.json (cli.cpp:35-131).

Counters, creation log, byte classes and snapshot files are identical to the
reference's for the same scenario (tests/test_output_path.py); the timing
columns are this engine's own wall-clock.  `workers` is reported as the
reference would (one per device) — there are no CPU worker threads here.
"""
from __future__ import annotations

import dataclasses
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


# ---- compare mode (proj/src/cli.cpp:133-157) --------------------------------
def _fmt_g(v: float, p: int) -> str:
    return "%.*g" % (p, v)


def _snapshot_diff(a_dir: str, b_dir: str, base: str) -> float:
    """max |a - b| over a snapshot pair (cli.cpp:20-31, read_raw dump.cpp:127)."""
    import numpy as np
    a = np.fromfile(os.path.join(a_dir, base + ".raw"), dtype="<f8")
    b = np.fromfile(os.path.join(b_dir, base + ".raw"), dtype="<f8")
    if a.size != b.size:
        raise RuntimeError("compare: snapshot size mismatch at " + base)
    return float(np.max(np.abs(a - b))) if a.size else 0.0


def run_compare(sc: S.Scenario, output_dir: str, iterations: int, name: str = "scenario",
                make_engine=None, **kw) -> dict:
    """`make_engine(scenario)` overrides the engine (tests pass the reference
    engine to check these writers against the reference's on CPU)."""
    def one(mode, sub):
        m = dataclasses.replace(sc, mode=mode)
        eng = make_engine(m) if make_engine else None
        try:
            return run_scenario(m, os.path.join(output_dir, sub), iterations, name=name, engine=eng, **kw)
        finally:
            if eng is not None:
                eng.close()
    st = one(S.MODE_STATIC, "static")
    pr = one(S.MODE_PROGRESSIVE, "progressive")
    diffs = [(b, _snapshot_diff(os.path.join(output_dir, "static"), os.path.join(output_dir, "progressive"), b))
             for b in pr["snapshot_bases"]]
    dmax = max([d for _, d in diffs], default=0.0)
    # compare.csv (cli.cpp:33-82): footprint = tile_footprint_bytes (tile.cpp:7-13)
    g = sc.tile_extent + 2
    fp = g * g * g * (sc.n_components * (2 * 19 + 8) * 8 + 1)
    at = {}
    for b, d in diffs:
        it = int(b[b.rfind("_i") + 2:])
        at[it] = max(at.get(it, d), d)
    cols = ["iteration"]
    for side in ("static", "progressive"):
        cols += [side + c for c in ("_tiles", "_active_cells", "_resident_bytes", "_bytes_intra",
                                    "_bytes_p2p", "_bytes_staged", "_window_mlups", "_window_mlups_bbox")]
    lines = [",".join(cols + ["field_diff_max"])]
    for rs, rp in zip(st["rows"], pr["rows"]):
        f = [str(rs["iteration"])]
        for r in (rs, rp):
            f += [str(r["tiles"]), str(r["active_cells"]), str(r["tiles"] * fp)] + [str(v) for v in r["bytes"]]
            f += [_fmt_g(r["window_mlups"], 6), _fmt_g(r["window_mlups_bbox"], 6)]
        f.append(_fmt_g(at[rs["iteration"]], 17) if rs["iteration"] in at else "")
        lines.append(",".join(f))
    with open(os.path.join(output_dir, "compare.csv"), "w", newline="\n") as fh:
        fh.write("\n".join(lines) + "\n")
    # compare_summary.json (cli.cpp:84-131)
    out = ["{", '  "scenario": "%s",' % name]
    for key, r in (("static", st), ("progressive", pr)):
        s = r["summary"]
        out.append('  "%s": {"status": "%s", "iterations": %d, "tiles_final": %d, "peak_resident_bytes": %d, '
                   '"mlups": %s, "mlups_bbox": %s, "bytes_intra": %d, "bytes_p2p": %d, "bytes_staged": %d},'
                   % (key, s["status"], s["iterations"], s["tiles_final"], s["peak_resident_bytes"],
                      _fmt_g(s["mlups"], 6), _fmt_g(s["mlups_bbox"], 6), s["bytes"]["intra"],
                      s["bytes"]["p2p"], s["bytes"]["staged"]))
    ps, ss = pr["summary"]["peak_resident_bytes"], st["summary"]["peak_resident_bytes"]
    out.append('  "peak_bytes_ratio": %s,' % _fmt_g(ps / ss if ss else 0.0, 6))
    out.append('  "snapshot_diffs": [%s],' % ", ".join('{"base": "%s", "max": %s}' % (b, _fmt_g(d, 17))
                                                       for b, d in diffs))
    out.append('  "field_diff_max": %s' % _fmt_g(dmax, 17))
    with open(os.path.join(output_dir, "compare_summary.json"), "w", newline="\n") as fh:
        fh.write("\n".join(out) + "\n}\n")
    return {"static_run": st, "progressive_run": pr, "diffs": diffs, "max_abs_diff": dmax}
