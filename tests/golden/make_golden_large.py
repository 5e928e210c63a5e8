"""Golden states at BASELINE.json scale, produced by the REFERENCE itself
(oracle/_ref/libplbm_ref.so, compiled from /root/reference/proj/src by
oracle/Makefile).  Run in the build container (the reference sources are not
on the GPU box; the fixture travels with the repo):

    python tests/golden/make_golden_large.py [name ...]

Scenarios (tests/test_gpu_large.py replays them on the GPU):
  c1_exact   BASELINE configs[0] exactly: D3Q19 single-component ideal gas,
             moving inflow box into 64^3, 16^3 subdomains, progressive
             S = 1e-12, 500 steps
  c2_100     BASELINE configs[1] = the benchmark workload: two-component PR
             liquid/vapour + ideal-like sphere release, 256^3, 32^3
             subdomains, progressive S = 1e-9, 100 steps (504 of 512 tiles
             by then), owners placed over 16 simulated devices (the
             reference runs 16 worker threads on them; scenario.bench_c2)
Each entry: counters, creation log, tile list, and one SHA-256 per (tile,
component) over the raw little-endian float64 bytes of the fields f, rho,
ux, uy, uz, u_prev (x, y, z) and psi, in that order.
"""
import hashlib
import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from paper_1510_03560_b200 import capi  # noqa: E402
from paper_1510_03560_b200 import scenario as S  # noqa: E402
from tests.compare import FIELDS  # noqa: E402

OUT = os.path.join(HERE, "large_states.json")


def c1_exact():
    return S.config1(threshold=1e-12), 500, 1


def c2_100():
    return S.bench_c2(), 100, 16


LARGE = {"c1_exact": c1_exact, "c2_100": c2_100}


def tile_digests(eng):
    sc = eng.scenario
    out = {}
    for coords, _, _ in eng.tiles():
        for c in range(sc.n_components):
            h = hashlib.sha256()
            for f in FIELDS:
                h.update(eng.read_tile(coords, c, f).astype("<f8").tobytes())
            out[f"{coords[0]},{coords[1]},{coords[2]}|{c}"] = h.hexdigest()
    return out


def summary(eng):
    d = {"counters": eng.counters(), "creation_log": eng.creation_log(), "tiles": eng.tiles(),
         "digests": tile_digests(eng)}
    return json.loads(json.dumps(d))  # tuples -> lists


def main(names):
    res = json.load(open(OUT)) if os.path.exists(OUT) else {}
    for name in names:
        sc, steps, workers = LARGE[name]()
        t0 = time.time()
        eng = capi.ref_engine(sc, workers=workers)
        eng.step(steps)
        res[name] = {"steps": steps, **summary(eng)}
        eng.close()
        print(name, res[name]["counters"]["tiles"], "tiles", f"{time.time() - t0:.0f} s", flush=True)
        with open(OUT, "w") as fh:
            json.dump(res, fh, indent=0, sort_keys=True)


if __name__ == "__main__":
    main(sys.argv[1:] or list(LARGE))
