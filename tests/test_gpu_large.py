"""Parity at BASELINE.json scale: the GPU engine against golden states the
REFERENCE produced at the benchmark's own shapes (tests/golden/
make_golden_large.py, oracle/_ref built from /root/reference/proj/src):

  c1_exact  configs[0] exactly (64^3, 16^3 tiles, 1 component, S = 1e-12,
            500 steps)
  c2_100    configs[1] = the bench workload (256^3, 32^3 tiles, 2-component
            MPMC, S = 1e-9, 100 steps: 504 of 512 tiles, the mesh the timed
            steps run on), owners over 8 simulated devices

Bit-exact: counters (iteration, cell updates, diagnostics, byte classes,
suppressed expansions), the creation log (activation set, order, trigger
face, owner) and a SHA-256 per (tile, component) over every field (f, rho, u,
u_prev, psi)."""
import json
import os

import pytest

from paper_1510_03560_b200 import capi
from tests.golden.make_golden_large import LARGE, OUT, summary

pytestmark = pytest.mark.gpu


def _golden():
    with open(OUT) as fh:
        return json.load(fh)


@pytest.mark.parametrize("name", sorted(LARGE))
def test_gpu_matches_reference_at_baseline_scale(built, name):
    g = _golden()[name]
    sc, steps, _ = LARGE[name]()
    assert steps == g["steps"]
    gpu = capi.gpu_engine(sc, capture=True)
    gpu.step(steps)
    d = summary(gpu)
    assert d["counters"] == g["counters"], (d["counters"], g["counters"])
    assert d["creation_log"] == g["creation_log"]
    assert d["tiles"] == g["tiles"]
    bad = [k for k in g["digests"] if d["digests"].get(k) != g["digests"][k]]
    assert not bad, f"{len(bad)} of {len(g['digests'])} (tile, component) states differ, e.g. {bad[:5]}"
