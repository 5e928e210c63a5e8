"""Output path: snapshots and report files of the B200 engine
against the reference's own writers.

* dump_field: the GPU engine's <base>.raw/.meta/.pgm must equal, byte for byte,
  the files iobench::dump_field (proj/src/dump.cpp:59-125) writes from the
  reference engine's state after the same steps (rho, u_magnitude, psi).
The report files of a whole run (engine::run_scenario, compare mode) are
checked through the C++ driver that links the reference's own writers
(tests/test_integration_driver.py).
"""
import pytest

from paper_1510_03560_b200 import capi
from tests import scenarios
from tests.conftest import have_ref

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
