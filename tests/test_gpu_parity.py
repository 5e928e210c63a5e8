"""GPU parity: the B200 engine (through the C-ABI) against the oracle
restatement, bit for bit in FP64 — every field of every tile, the creation
log (activation set + order + trigger + owner), the diagnostics counters and
the modeled byte classes."""
import pytest

from paper_1510_03560_b200 import capi
from tests import scenarios
from tests.compare import assert_same_state

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("variant", [0, 1, 2, 22, 100, 200], ids=["default_percomp", "plain", "tmem_both_comps", "percomp_lag2", "percomp_fused_face", "percomp_strided_xfaces"])
@pytest.mark.parametrize("name", sorted(scenarios.ALL))
def test_gpu_matches_oracle(built, name, variant):
    make, steps = scenarios.ALL[name]
    sc = make()
    orc = capi.oracle_engine(sc)
    gpu = capi.gpu_engine(sc, capture=True)
    gpu.set_kernel_variant(variant)
    assert_same_state(orc, gpu, label=f"{name}@0")
    orc.step(1)
    gpu.step(1)
    assert_same_state(orc, gpu, label=f"{name}@1")
    orc.step(steps - 1)
    gpu.step(steps - 1)
    assert_same_state(orc, gpu, label=f"{name}@{steps}")


@pytest.mark.parametrize("name", sorted(__import__("tests.golden_check", fromlist=["x"]).load_golden()))
def test_gpu_reproduces_reference_golden_states(built, name):
    """Against the state the reference itself produced (tests/golden/)."""
    from tests.golden_check import assert_matches_golden
    make, steps = scenarios.ALL[name]
    gpu = capi.gpu_engine(make(), capture=True)
    gpu.step(steps)
    assert_matches_golden(gpu, name)
