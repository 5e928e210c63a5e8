"""Bitwise state comparison between two engines behind the step-loop C-ABI."""
import numpy as np

from paper_1510_03560_b200 import scenario as S

FIELDS = (S.FIELD_F, S.FIELD_RHO, S.FIELD_UX, S.FIELD_UY, S.FIELD_UZ,
          S.FIELD_PUX, S.FIELD_PUY, S.FIELD_PUZ, S.FIELD_PSI)


def assert_same_state(a, b, fields=FIELDS, label=""):
    ca, cb = a.counters(), b.counters()
    assert ca == cb, f"{label} counters differ:\n{ca}\n{cb}"
    assert a.creation_log() == b.creation_log(), f"{label} creation logs differ"
    ta = a.tiles()
    assert ta == b.tiles(), f"{label} tile sets differ"
    bad = []
    for (coords, _owner, _birth) in ta:
        for comp in range(a.scenario.n_components):
            for fld in fields:
                x = a.read_tile(coords, comp, fld)
                y = b.read_tile(coords, comp, fld)
                if not np.array_equal(x.view(np.uint64), y.view(np.uint64)):
                    diff = np.abs(x - y)
                    bad.append((coords, comp, fld, int(np.count_nonzero(x.view(np.uint64) != y.view(np.uint64))),
                                float(np.nanmax(diff))))
    assert not bad, f"{label} {len(bad)} field mismatches, first: {bad[:6]}"
