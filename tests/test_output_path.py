"""Output path: snapshots and report files of the B200 engine
against the reference's own writers.

* dump_field: the GPU engine's <base>.raw/.meta/.pgm must equal, byte for byte,
  the files iobench::dump_field (proj/src/dump.cpp:59-125) writes from the
  reference engine's state after the same steps (rho, u_magnitude, psi).
* run_scenario: paper_1510_03560_b200.driver against engine::run_scenario
  (proj/src/engine.cpp:580-704) — creation_log.csv identical, time_series.csv
  and summary.json identical except the wall-clock columns, snapshots identical.
"""
import csv
import json
import os

import pytest

from paper_1510_03560_b200 import capi, driver
from tests import scenarios
from tests.conftest import have_ref

TIMING_COLS = {"window_seconds", "window_mlups", "window_mlups_bbox"}
TIMING_KEYS = {"compute_seconds", "mlups", "mlups_bbox", "name", "workers"}


def test_driver_writers_format(tmp_path):
    """Writers alone (no GPU): header lines and JSON layout."""
    driver._write_creation_log([(0, (1, 2, 3), "init", 0), (5, (2, 2, 3), "+x", 1)],
                               str(tmp_path / "c.csv"))
    assert (tmp_path / "c.csv").read_text() == (
        "iteration,tile_x,tile_y,tile_z,trigger_face,owner_device\n0,1,2,3,init,0\n5,2,2,3,+x,1\n")
    driver._write_time_series([{"iteration": 10, "tiles": 3, "active_cells": 4, "bytes": [1, 2, 3],
                                "window_seconds": 0.5, "window_mlups": 0.1, "window_mlups_bbox": 2.0,
                                "window_negative_populations": 0, "window_psi_clamps": 1,
                                "window_suppressed_expansions": 2}], str(tmp_path / "t.csv"))
    rows = list(csv.reader(open(tmp_path / "t.csv")))
    assert rows[1] == ["10", "3", "4", "1", "2", "3", "0.5", "0.10000000000000001", "2", "0", "1", "2"]


def _files_equal(a, b):
    return open(a, "rb").read() == open(b, "rb").read()


@pytest.mark.gpu
@pytest.mark.skipif(not have_ref(), reason="reference shim not built")
@pytest.mark.parametrize("name", ["mpmc_progressive_e16", "mpmc_e32_solid_periodic", "c1_progressive"])
def test_dump_field_matches_reference(built, tmp_path, name):
    make, steps = scenarios.ALL[name]
    sc = make()
    ref = capi.ref_engine(sc)
    gpu = capi.gpu_engine(sc, capture=True)
    ref.step(steps)
    gpu.step(steps)
    for field in ("rho", "u_magnitude", "psi"):
        for c in range(sc.n_components):
            a, b = str(tmp_path / f"g_{field}_{c}"), str(tmp_path / f"r_{field}_{c}")
            gpu.dump_field(field, c, steps, a, True)
            ref.dump_field(field, c, steps, b, True)
            for ext in (".raw", ".meta", ".pgm"):
                assert _files_equal(a + ext, b + ext), (field, c, ext)


@pytest.mark.gpu
@pytest.mark.skipif(not have_ref(), reason="reference shim not built")
def test_run_scenario_matches_reference_driver(built, tmp_path):
    make, steps = scenarios.ALL["mpmc_progressive_e16"]
    sc = make()
    kw = dict(iterations=steps, report_interval=4, snapshot_interval=5, with_pgm=True)
    ref_dir, gpu_dir = str(tmp_path / "ref"), str(tmp_path / "gpu")
    capi.ref_run_scenario(sc, ref_dir, fields=("rho", "psi"), name="t", **kw)
    driver.run_scenario(sc, gpu_dir, steps, report_interval=4, snapshot_interval=5,
                        snapshot_fields=("rho", "psi"), snapshot_pgm=True, name="t")
    assert _files_equal(f"{ref_dir}/creation_log.csv", f"{gpu_dir}/creation_log.csv")
    ra = list(csv.DictReader(open(f"{ref_dir}/time_series.csv")))
    ga = list(csv.DictReader(open(f"{gpu_dir}/time_series.csv")))
    assert len(ra) == len(ga)
    for r, g in zip(ra, ga):
        assert {k: v for k, v in r.items() if k not in TIMING_COLS} == \
               {k: v for k, v in g.items() if k not in TIMING_COLS}
    rs, gs = json.load(open(f"{ref_dir}/summary.json")), json.load(open(f"{gpu_dir}/summary.json"))
    assert sorted(rs) == sorted(gs)
    assert {k: v for k, v in rs.items() if k not in TIMING_KEYS} == \
           {k: v for k, v in gs.items() if k not in TIMING_KEYS}
    snaps = sorted(os.listdir(f"{ref_dir}/snapshots"))
    assert snaps == sorted(os.listdir(f"{gpu_dir}/snapshots"))
    for f in snaps:
        assert _files_equal(f"{ref_dir}/snapshots/{f}", f"{gpu_dir}/snapshots/{f}"), f
