"""Generates tests/golden/golden_states.json from the REFERENCE itself
(oracle/_ref/libplbm_ref.so, compiled from /root/reference/proj/src by
oracle/Makefile).  Run in the build container (the reference sources are not
on the GPU box; the fixture travels with the repo):

    python tests/golden/make_golden.py

Each entry: the scenario name, step count, counters, creation log, tile list
and a SHA-256 of every field (f, rho, u, u_prev, psi) of every tile/component
after the steps, as raw little-endian float64 bytes.
"""
import hashlib
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from paper_1510_03560_b200 import capi  # noqa: E402
from tests import scenarios  # noqa: E402
from tests.compare import FIELDS  # noqa: E402

GOLDEN = ["c1_progressive", "c1_progressive_S0", "mpmc_progressive_e16", "mpmc_e32",
          "periodic_solid_gravity", "mpmc_e16_solid_S0", "mpmc_islands", "mpmc_e64", "mpmc3_e64_solid",
          "mp1_e16", "mp1_e32_solid", "mpmc3_e16"]


def state_digest(eng):
    sc = eng.scenario
    out = {"counters": eng.counters(), "creation_log": eng.creation_log(),
           "tiles": eng.tiles(), "fields": {}}
    for coords, _, _ in out["tiles"]:
        for c in range(sc.n_components):
            for f in FIELDS:
                a = eng.read_tile(coords, c, f)
                key = f"{coords[0]},{coords[1]},{coords[2]}|{c}|{f}"
                out["fields"][key] = hashlib.sha256(a.astype("<f8").tobytes()).hexdigest()
    out["counters"]["bytes"] = list(out["counters"]["bytes"])
    out["creation_log"] = [list(map(lambda v: list(v) if isinstance(v, tuple) else v, r))
                           for r in out["creation_log"]]
    out["tiles"] = [[list(c), o, b] for c, o, b in out["tiles"]]
    return out


def main():
    res = {}
    for name in GOLDEN:
        make, steps = scenarios.ALL[name]
        eng = capi.ref_engine(make(), workers=4)
        eng.step(steps)
        res[name] = {"steps": steps, **state_digest(eng)}
        eng.close()
        print(name, res[name]["counters"]["tiles"], "tiles")
    with open(os.path.join(HERE, "golden_states.json"), "w") as fh:
        json.dump(res, fh, indent=0, sort_keys=True)


if __name__ == "__main__":
    main()
