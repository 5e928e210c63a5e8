"""The oracle restatement (oracle/plbm_oracle.c) is pinned bit-for-bit against
the reference engine itself (oracle/_ref/libplbm_ref.so, built from
/root/reference/proj/src by oracle/Makefile)."""
import pytest

from paper_1510_03560_b200 import capi
from tests import scenarios
from tests.compare import assert_same_state
from tests.conftest import have_ref

pytestmark = pytest.mark.skipif(not have_ref(), reason="reference shim not built")


@pytest.mark.parametrize("name", sorted(scenarios.ALL))
def test_oracle_matches_reference(built, name):
    make, steps = scenarios.ALL[name]
    sc = make()
    ref = capi.ref_engine(sc, workers=4)
    orc = capi.oracle_engine(sc)
    assert_same_state(ref, orc, label=f"{name}@0")
    ref.step(steps)
    orc.step(steps)
    assert_same_state(ref, orc, label=f"{name}@{steps}")
