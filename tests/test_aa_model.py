"""CPU model of the A-A storage rules (csrc/kernels.cuh AA_LOCAL / AA_NEIGH)
against the A-B pull they replace, on a small 2-D-in-3-D D3Q19 grid with
solids: one tile, periodic or bounded, arbitrary post-collision values.

* ownership: in each step kind every storage location (cell, direction) of a
  fluid cell is read by at most one cell and written by at most one cell, and
  when both happen it is the same cell (so the in-place update is race-free
  under any schedule, given that a cell reads before it writes);
* equivalence: two A-A steps (LOCAL then NEIGH) deliver, to every fluid cell,
  exactly the f_in the A-B pull rule delivers from the same post-collision
  values (f_in[i](x) = solid(x - e_i) ? f_post(x)[opp i] : f_post(x - e_i)[i]),
  and likewise NEIGH then LOCAL."""
import itertools

import numpy as np

EX = [0, 1, -1, 0, 0, 0, 0, 1, -1, 1, -1, 1, -1, 1, -1, 0, 0, 0, 0]
EY = [0, 0, 0, 1, -1, 0, 0, 1, -1, -1, 1, 0, 0, 0, 0, 1, -1, 1, -1]
EZ = [0, 0, 0, 0, 0, 1, -1, 0, 0, 0, 0, 1, -1, -1, 1, 1, -1, -1, 1]
OPP = [0, 2, 1, 4, 3, 6, 5, 8, 7, 10, 9, 12, 11, 14, 13, 16, 15, 18, 17]
Q = 19
N = 6


def _setup(seed):
    rng = np.random.default_rng(seed)
    solid = rng.random((N, N, N)) < 0.2
    cells = [c for c in itertools.product(range(N), repeat=3) if not solid[c]]
    sh = lambda c, i, s: ((c[0] + s * EX[i]) % N, (c[1] + s * EY[i]) % N, (c[2] + s * EZ[i]) % N)  # periodic
    return rng, solid, cells, sh


def _aa_reads_writes(kind, c, solid, sh):
    """Locations cell c reads (per direction i: where f_in[i] comes from) and
    writes (per direction i: where f_post[i] goes) in one step of `kind`."""
    reads, writes = {}, {}
    for i in range(Q):
        src = sh(c, i, -1)
        if kind == "local":
            reads[i] = (c, i)
            writes[i] = (c, OPP[i])
        else:
            reads[i] = (c, i) if solid[src] else (src, OPP[i])
            dst = sh(c, i, +1)
            writes[i] = (c, OPP[i]) if solid[dst] else (dst, i)
    return reads, writes


def test_aa_ownership_is_exclusive():
    for seed in range(5):
        _, solid, cells, sh = _setup(seed)
        for kind in ("local", "neigh"):
            reader, writer = {}, {}
            for c in cells:
                r, w = _aa_reads_writes(kind, c, solid, sh)
                for loc in r.values():
                    assert loc not in reader, (kind, loc)
                    reader[loc] = c
                for loc in w.values():
                    assert loc not in writer, (kind, loc)
                    writer[loc] = c
            for loc, c in reader.items():
                assert writer.get(loc, c) == c, (kind, loc)
            for loc in writer:
                assert not solid[loc[0]], (kind, loc)  # solid cells' storage is never touched


def _ab_pull(fpost, c, solid, sh):
    return [fpost[c][OPP[i]] if solid[sh(c, i, -1)] else fpost[sh(c, i, -1)][i] for i in range(Q)]


def test_aa_two_steps_equal_ab_pull():
    for seed in range(5):
        rng, solid, cells, sh = _setup(seed)
        for first, second in (("local", "neigh"), ("neigh", "local")):
            store = {}
            # state before `first` reads: produce it by applying the previous
            # kind's writes to arbitrary post-collision values g
            prev = "neigh" if first == "local" else "local"
            g = {c: rng.random(Q) for c in cells}
            for c in cells:
                _, w = _aa_reads_writes(prev, c, solid, sh)
                for i, loc in w.items():
                    store[loc] = g[c][i]
            # `first` step: every cell must read exactly the A-B pull of g
            fpost = {c: rng.random(Q) for c in cells}
            for c in cells:
                r, _ = _aa_reads_writes(first, c, solid, sh)
                assert [store[r[i]] for i in range(Q)] == list(_ab_pull(g, c, solid, sh))
            for c in cells:  # reads all happen-before writes per cell (any order across cells)
                _, w = _aa_reads_writes(first, c, solid, sh)
                for i, loc in w.items():
                    store[loc] = fpost[c][i]
            for c in cells:
                r, _ = _aa_reads_writes(second, c, solid, sh)
                assert [store[r[i]] for i in range(Q)] == list(_ab_pull(fpost, c, solid, sh))
