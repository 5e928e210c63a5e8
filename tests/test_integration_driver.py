"""The reference's C++ driver on the B200 engine (integration/plbm_gpu_run.cpp,
SURVEY §8(b) "C++ side"): the same scenario TOML through the reference's own
loader, run by engine::run_scenario (the reference) and by plbm_gpu_run (the
GPU engine behind the C-ABI, the reference's report writers) -> identical
creation_log.csv, time_series.csv and summary.json except the wall-clock
fields, and identical snapshot files."""
import csv
import ctypes as C
import json
import os
import subprocess

import pytest

from paper_1510_03560_b200 import capi
from tests import scenarios
from tests.conftest import have_ref

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(REPO, "integration", "_bin", "plbm_gpu_run")
TIMING_COLS = {"window_seconds", "window_mlups", "window_mlups_bbox"}
TIMING_KEYS = {"compute_seconds", "mlups", "mlups_bbox"}

pytestmark = pytest.mark.skipif(not have_ref(), reason="reference shim not built")


def ref_run_toml(path, out):
    lib = capi.load(capi.REF_LIB, "plbm_ref")
    lib.plbm_ref_run_toml.restype = C.c_int
    lib.plbm_ref_run_toml.argtypes = [C.c_char_p, C.c_char_p]
    assert lib.plbm_ref_run_toml(path.encode(), out.encode()) == 0


def assert_same_outputs(a, b):
    assert open(f"{a}/creation_log.csv").read() == open(f"{b}/creation_log.csv").read()
    ra = list(csv.DictReader(open(f"{a}/time_series.csv")))
    rb = list(csv.DictReader(open(f"{b}/time_series.csv")))
    assert len(ra) == len(rb) > 0
    for x, y in zip(ra, rb):
        assert {k: v for k, v in x.items() if k not in TIMING_COLS} == \
               {k: v for k, v in y.items() if k not in TIMING_COLS}
    sa, sb = json.load(open(f"{a}/summary.json")), json.load(open(f"{b}/summary.json"))
    assert sorted(sa) == sorted(sb)
    assert {k: v for k, v in sa.items() if k not in TIMING_KEYS} == \
           {k: v for k, v in sb.items() if k not in TIMING_KEYS}
    if os.path.isdir(f"{a}/snapshots"):
        names = sorted(os.listdir(f"{a}/snapshots"))
        assert names == sorted(os.listdir(f"{b}/snapshots"))
        for n in names:
            assert open(f"{a}/snapshots/{n}", "rb").read() == open(f"{b}/snapshots/{n}", "rb").read(), n


def test_toml_writer_round_trips_through_the_reference_loader(built, tmp_path):
    """Scenario.to_toml -> iobench::load_config gives the run the descriptor
    gives (both on the reference)."""
    make, steps = scenarios.ALL["c1_progressive"]
    sc = make()
    toml = str(tmp_path / "s.toml")
    sc.to_toml(toml, iterations=steps, report_interval=5, snapshot_interval=10)
    ref_run_toml(toml, str(tmp_path / "a"))
    capi.ref_run_scenario(sc, str(tmp_path / "b"), iterations=steps, report_interval=5,
                          snapshot_interval=10, name=sc.name)
    assert_same_outputs(str(tmp_path / "a"), str(tmp_path / "b"))


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["mpmc_progressive_e16", "mpmc_channel_e16"])
def test_cpp_driver_matches_reference_driver(built, tmp_path, name):
    make, steps = scenarios.ALL[name]
    sc = make()
    toml = str(tmp_path / "s.toml")
    sc.to_toml(toml, iterations=steps, report_interval=4, snapshot_interval=5,
               snapshot_fields=("rho", "u_magnitude", "psi"), snapshot_pgm=True)
    ref_run_toml(toml, str(tmp_path / "ref"))
    r = subprocess.run([BIN, toml, "--output", str(tmp_path / "gpu")], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    assert_same_outputs(str(tmp_path / "ref"), str(tmp_path / "gpu"))


# ---- compare mode (proj/src/cli.cpp:133-157) ---------------------------------
def ref_run_compare_toml(path, out):
    lib = capi.load(capi.REF_LIB, "plbm_ref")
    lib.plbm_ref_run_compare_toml.restype = C.c_int
    lib.plbm_ref_run_compare_toml.argtypes = [C.c_char_p, C.c_char_p]
    assert lib.plbm_ref_run_compare_toml(path.encode(), out.encode()) == 0


def assert_same_compare(a, b):
    """compare.csv / compare_summary.json equal except the wall-clock
    columns; both runs' own outputs equal as in assert_same_outputs."""
    for side in ("static", "progressive"):
        assert_same_outputs(f"{a}/{side}", f"{b}/{side}")
    ra = list(csv.DictReader(open(f"{a}/compare.csv")))
    rb = list(csv.DictReader(open(f"{b}/compare.csv")))
    assert open(f"{a}/compare.csv").readline() == open(f"{b}/compare.csv").readline()
    assert len(ra) == len(rb) > 0
    timing = {s + c for s in ("static", "progressive") for c in ("_window_mlups", "_window_mlups_bbox")}
    for x, y in zip(ra, rb):
        assert {k: v for k, v in x.items() if k not in timing} == {k: v for k, v in y.items() if k not in timing}
    assert any(r["field_diff_max"] for r in ra)
    sa, sb = json.load(open(f"{a}/compare_summary.json")), json.load(open(f"{b}/compare_summary.json"))
    for s in (sa, sb):
        for side in ("static", "progressive"):
            s[side].pop("mlups"), s[side].pop("mlups_bbox")
    assert sa == sb
    assert len(sa["snapshot_diffs"]) > 0


def _compare_toml(tmp_path, name):
    make, steps = scenarios.ALL[name]
    sc = make()
    toml = str(tmp_path / "s.toml")
    sc.to_toml(toml, iterations=steps, report_interval=4, snapshot_interval=5,
               snapshot_fields=("rho", "psi"), snapshot_pgm=True)
    return sc, steps, toml


@pytest.mark.gpu
def test_compare_mode_matches_reference(built, tmp_path):
    sc, steps, toml = _compare_toml(tmp_path, "mpmc_channel_e16")
    ref_run_compare_toml(toml, str(tmp_path / "ref"))
    out = str(tmp_path / "gpu")
    r = subprocess.run([BIN, toml, "--output", out, "--compare", "1"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    assert_same_compare(str(tmp_path / "ref"), out)
