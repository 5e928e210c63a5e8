/*
 * plbm_oracle.c — CPU restatement of the reference step loop.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the B200
 * engine: only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline
 * leg may load it.  The product path (libplbm_gpu.so) never links or calls
 * it, and there is no CPU fallback anywhere in the product.
 *
 * It restates, single-threaded and in plain C, the algorithm of
 * /root/reference/proj (D3Q19 only), following its operation order exactly
 * so results are bit-identical (compiled with -ffp-contract=off, no -march).
 * Parity of this restatement is PINNED against the reference itself
 * (oracle/_ref/libplbm_ref.so, built from the reference sources by
 * oracle/Makefile) in tests/test_oracle.py, and against the reference's own
 * known-answer values in tests/test_golden.py.
 *
 * Every function cites the reference file:line it restates.
 */
#include "plbm_scenario.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define Q 19

/* proj/src/stencil.cpp:21-34 — D3Q19 velocity order and weights. */
static const int E3[Q][3] = {
    {0, 0, 0},
    {1, 0, 0},  {-1, 0, 0}, {0, 1, 0},  {0, -1, 0}, {0, 0, 1},  {0, 0, -1},
    {1, 1, 0},  {-1, -1, 0}, {1, -1, 0}, {-1, 1, 0},
    {1, 0, 1},  {-1, 0, -1}, {1, 0, -1}, {-1, 0, 1},
    {0, 1, 1},  {0, -1, -1}, {0, 1, -1}, {0, -1, 1},
};
static const double W3[Q] = {
    1.0 / 3.0,
    1.0 / 18.0, 1.0 / 18.0, 1.0 / 18.0, 1.0 / 18.0, 1.0 / 18.0, 1.0 / 18.0,
    1.0 / 36.0, 1.0 / 36.0, 1.0 / 36.0, 1.0 / 36.0,
    1.0 / 36.0, 1.0 / 36.0, 1.0 / 36.0, 1.0 / 36.0,
    1.0 / 36.0, 1.0 / 36.0, 1.0 / 36.0, 1.0 / 36.0,
};
static int OPP[Q];
static const double CS2 = 1.0 / 3.0; /* proj/include/plbm/stencil.hpp:20 */

/* proj/src/stencil.cpp:57-69 — opp derived by search. */
static void init_opp(void) {
    for (int i = 0; i < Q; ++i)
        for (int j = 0; j < Q; ++j)
            if (E3[j][0] == -E3[i][0] && E3[j][1] == -E3[i][1] &&
                E3[j][2] == -E3[i][2]) {
                OPP[i] = j;
                break;
            }
}

/* ---------------------------------------------------------------- L0 */

/* proj/include/plbm/kernels.hpp:17-28 */
static void equilibrium(double rho, const double u[3], double* out) {
    const double uu = u[0] * u[0] + u[1] * u[1] + u[2] * u[2];
    const double inv_cs2 = 1.0 / CS2;
    for (int i = 0; i < Q; ++i) {
        const double eu = (double)E3[i][0] * u[0] + (double)E3[i][1] * u[1] +
                          (double)E3[i][2] * u[2];
        out[i] = W3[i] * rho *
                 (1.0 + eu * inv_cs2 + 0.5 * eu * eu * inv_cs2 * inv_cs2 -
                  0.5 * uu * inv_cs2);
    }
}

/* proj/include/plbm/kernels.hpp:31-48 */
static void moments(const double* f, double* rho_out, double u[3]) {
    double rho = 0.0, m0 = 0.0, m1 = 0.0, m2 = 0.0;
    for (int i = 0; i < Q; ++i) {
        rho += f[i];
        m0 += f[i] * (double)E3[i][0];
        m1 += f[i] * (double)E3[i][1];
        m2 += f[i] * (double)E3[i][2];
    }
    if (rho != 0.0) {
        u[0] = m0 / rho;
        u[1] = m1 / rho;
        u[2] = m2 / rho;
    } else {
        u[0] = u[1] = u[2] = 0.0;
    }
    *rho_out = rho;
}

/* proj/src/kernels.cpp:5-30 — pull streaming with half-way bounce-back. */
static void stream_pull(const double* f_read, double* f_write,
                        const unsigned char* solid, int g) {
    const size_t gcells = (size_t)g * g * g;
    for (int i = 0; i < Q; ++i) {
        const long shift = E3[i][0] + (long)g * (E3[i][1] + (long)g * E3[i][2]);
        const double* src = f_read + (size_t)i * gcells;
        const double* rev = f_read + (size_t)OPP[i] * gcells;
        double* dst = f_write + (size_t)i * gcells;
        for (int z = 1; z < g - 1; ++z)
            for (int y = 1; y < g - 1; ++y) {
                const long row = (long)g * (y + (long)g * z);
                for (int x = 1; x < g - 1; ++x) {
                    const long c = row + x;
                    if (solid[c]) continue;
                    const long from = c - shift;
                    dst[c] = solid[from] ? rev[c] : src[from];
                }
            }
    }
}

/* ---------------------------------------------------------------- L1 */

/* proj/src/physics.cpp:12-27 — returns 0, or 1 at the b*rho >= 1 pole. */
static int pr_pressure(double rho, const plbm_component_desc* p, double* out) {
    if (p->b * rho >= 1.0) return 1;
    double theta = 1.0;
    if (p->Tc > 0.0) {
        const double kappa =
            0.37464 + 1.54226 * p->omega - 0.26992 * p->omega * p->omega;
        const double root = 1.0 + kappa * (1.0 - sqrt(p->T / p->Tc));
        theta = root * root;
    }
    const double ideal = rho * p->R * p->T / (1.0 - p->b * rho);
    const double attr = p->a * theta * rho * rho /
                        (1.0 + 2.0 * p->b * rho - p->b * p->b * rho * rho);
    *out = ideal - attr;
    return 0;
}

/* proj/src/physics.cpp:34-42 */
static double pseudo_potential(double rho, double press, double g_self,
                               unsigned long long* clamps) {
    const double radicand = 2.0 * (press - CS2 * rho) / (CS2 * g_self);
    if (radicand < 0.0) {
        if (clamps) ++*clamps;
        return 0.0;
    }
    return sqrt(radicand);
}

/* proj/src/physics.cpp:44-63 */
static void intra_force(const double* psi, long cell, const long stride[3],
                        const plbm_component_desc* p, double F[3]) {
    double s1[3] = {0, 0, 0}, s2[3] = {0, 0, 0};
    for (int i = 1; i < Q; ++i) {
        const long n = cell + E3[i][0] * stride[0] + E3[i][1] * stride[1] +
                       E3[i][2] * stride[2];
        const double pn = psi[n];
        const double w = W3[i];
        for (int d = 0; d < 3; ++d) {
            s1[d] += w * pn * (double)E3[i][d];
            s2[d] += w * pn * pn * (double)E3[i][d];
        }
    }
    const double c1 = -p->beta * p->g_self * psi[cell];
    const double c2 = -0.5 * (1.0 - p->beta) * p->g_self;
    for (int d = 0; d < 3; ++d) F[d] = c1 * s1[d] + c2 * s2[d];
}

/* proj/src/physics.cpp:65-78 */
static void inter_force(double psi_self, const double* psi_other, long cell,
                        const long stride[3], double g_cross, double F[3]) {
    double s1[3] = {0, 0, 0};
    for (int i = 1; i < Q; ++i) {
        const long n = cell + E3[i][0] * stride[0] + E3[i][1] * stride[1] +
                       E3[i][2] * stride[2];
        const double w = W3[i];
        for (int d = 0; d < 3; ++d) s1[d] += w * psi_other[n] * (double)E3[i][d];
    }
    const double c = -g_cross * psi_self;
    for (int d = 0; d < 3; ++d) F[d] = c * s1[d];
}

/* ---------------------------------------------------------------- L2 */

typedef struct {
    int c[3];
    int owner;
    long birth;
    size_t log_index;
    int cur;
    double* f[2];                 /* [C][Q][gcells] each                   */
    double *rho, *ux, *uy, *uz;   /* [C][gcells]                           */
    double *pux, *puy, *puz, *psi;
    unsigned char* solid;         /* [gcells]                              */
    int* bcells;                  /* boundary fluid cells                  */
    int* icells;                  /* interior fluid cells                  */
    int nb, ni;
} Tile;

typedef struct {
    long iteration;
    int c[3];
    int trigger;
    int owner;
} LogRow;

typedef struct {
    int src[3];
    int face;
} Trigger;

typedef struct {
    /* configuration */
    int dom[3], E, g, C, mode, periodic[3], devices, policy;
    size_t gcells;
    double threshold, weight_p2p, weight_staged;
    plbm_component_desc comp[PLBM_MAX_COMP];
    double coupling[PLBM_MAX_COMP * PLBM_MAX_COMP];
    plbm_seed_desc seeds[PLBM_MAX_SEEDS];
    int n_seeds;
    unsigned char* geom; /* domain bytes, x-fastest */
    unsigned char* p2p;  /* devices^2 */
    int grid[3];
    /* ambient, proj/src/tilemap.cpp:13-28 */
    double amb_rho[PLBM_MAX_COMP], amb_psi[PLBM_MAX_COMP];
    double amb_feq[PLBM_MAX_COMP][Q];
    /* state */
    Tile** tiles; /* linear (x*GY + y)*GZ + z: lexicographic TileCoord order */
    int n_tiles;
    LogRow* log;
    size_t n_log, cap_log;
    unsigned long long suppressed, active_cells;
    unsigned long long* per_dev;
    unsigned long long bytes[3];
    unsigned long long face_xfer;
    long iteration;
    unsigned long long cell_updates;
    unsigned long long neg, clamps, zero_rho;
    /* error */
    int err;
    int err_tile[3];
    long err_it;
    char err_phase[8];
    char err_msg[160];
} Oracle;

static size_t lin(const Oracle* o, int x, int y, int z) {
    return ((size_t)x * o->grid[1] + y) * o->grid[2] + z;
}
static Tile* at(const Oracle* o, int x, int y, int z) {
    return o->tiles[lin(o, x, y, z)];
}
/* proj/include/plbm/tile.hpp:68-73 (3-D) */
static size_t gidx(const Oracle* o, int lx, int ly, int lz) {
    return (size_t)(lx + 1) + (size_t)o->g * ((size_t)(ly + 1) + (size_t)o->g * (size_t)(lz + 1));
}
static int geom_at(const Oracle* o, int x, int y, int z) {
    if (!o->geom) return 0;
    return o->geom[(size_t)x + (size_t)o->dom[0] * ((size_t)y + (size_t)o->dom[1] * (size_t)z)] != 0;
}

/* proj/src/tilemap.cpp:56-67 */
static int neighbor_coords(const Oracle* o, const int from[3], int face, int out[3]) {
    int c[3] = {from[0], from[1], from[2]};
    const int axis = face / 2;
    c[axis] += (face % 2) ? 1 : -1;
    if (c[axis] < 0 || c[axis] >= o->grid[axis]) {
        if (!o->periodic[axis]) return 0;
        c[axis] = (c[axis] + o->grid[axis]) % o->grid[axis];
    }
    out[0] = c[0]; out[1] = c[1]; out[2] = c[2];
    return 1;
}
static Tile* neighbor(const Oracle* o, const Tile* t, int face) {
    int nc[3];
    if (!neighbor_coords(o, t->c, face, nc)) return NULL;
    return at(o, nc[0], nc[1], nc[2]);
}

static void log_push(Oracle* o, LogRow r) {
    if (o->n_log == o->cap_log) {
        o->cap_log = o->cap_log ? 2 * o->cap_log : 64;
        o->log = (LogRow*)realloc(o->log, o->cap_log * sizeof(LogRow));
    }
    o->log[o->n_log++] = r;
}

/* proj/src/tilemap.cpp:83-175 */
static Tile* create_tile(Oracle* o, const int c[3], long iteration, int trigger) {
    if (c[0] < 0 || c[0] >= o->grid[0] || c[1] < 0 || c[1] >= o->grid[1] ||
        c[2] < 0 || c[2] >= o->grid[2]) {
        ++o->suppressed;
        return NULL;
    }
    Tile* t = (Tile*)calloc(1, sizeof(Tile));
    memcpy(t->c, c, sizeof t->c);
    t->birth = iteration;
    t->owner = -1;
    const size_t gc = o->gcells;
    const int E = o->E, C = o->C;
    t->solid = (unsigned char*)calloc(gc, 1);
    for (int lz = -1; lz <= E; ++lz)
        for (int ly = -1; ly <= E; ++ly)
            for (int lx = -1; lx <= E; ++lx) {
                int gg[3] = {c[0] * E + lx, c[1] * E + ly, c[2] * E + lz};
                int outside = 0;
                for (int ax = 0; ax < 3; ++ax)
                    if (gg[ax] < 0 || gg[ax] >= o->dom[ax]) {
                        if (o->periodic[ax]) gg[ax] = (gg[ax] + o->dom[ax]) % o->dom[ax];
                        else outside = 1;
                    }
                if (!outside && geom_at(o, gg[0], gg[1], gg[2]))
                    t->solid[gidx(o, lx, ly, lz)] = 1;
            }
    for (int b = 0; b < 2; ++b) {
        t->f[b] = (double*)malloc((size_t)C * Q * gc * sizeof(double));
        for (int k = 0; k < C; ++k)
            for (int i = 0; i < Q; ++i) {
                double* p = t->f[b] + ((size_t)k * Q + i) * gc;
                for (size_t cell = 0; cell < gc; ++cell) p[cell] = o->amb_feq[k][i];
            }
    }
    double** arrs[8] = {&t->rho, &t->ux, &t->uy, &t->uz, &t->pux, &t->puy, &t->puz, &t->psi};
    for (int a = 0; a < 8; ++a) *arrs[a] = (double*)calloc((size_t)C * gc, sizeof(double));
    for (int k = 0; k < C; ++k)
        for (size_t cell = 0; cell < gc; ++cell)
            if (!t->solid[cell]) t->rho[(size_t)k * gc + cell] = o->amb_rho[k];
    t->bcells = (int*)malloc((size_t)E * E * E * sizeof(int));
    t->icells = (int*)malloc((size_t)E * E * E * sizeof(int));
    for (int lz = 0; lz < E; ++lz)
        for (int ly = 0; ly < E; ++ly)
            for (int lx = 0; lx < E; ++lx) {
                const size_t cell = gidx(o, lx, ly, lz);
                if (t->solid[cell]) continue;
                const int boundary = lx == 0 || lx == E - 1 || ly == 0 ||
                                     ly == E - 1 || lz == 0 || lz == E - 1;
                if (boundary) t->bcells[t->nb++] = (int)cell;
                else t->icells[t->ni++] = (int)cell;
            }
    o->active_cells += (unsigned long long)(t->nb + t->ni);
    t->log_index = o->n_log;
    LogRow r = {iteration, {c[0], c[1], c[2]}, trigger, -1};
    log_push(o, r);
    o->tiles[lin(o, c[0], c[1], c[2])] = t;
    ++o->n_tiles;
    return t;
}

static void free_tile(Tile* t) {
    if (!t) return;
    free(t->f[0]); free(t->f[1]);
    free(t->rho); free(t->ux); free(t->uy); free(t->uz);
    free(t->pux); free(t->puy); free(t->puz); free(t->psi);
    free(t->solid); free(t->bcells); free(t->icells);
    free(t);
}

/* ---------------------------------------------------------------- L2' */

/* proj/src/topology.cpp:91-94 (0 intra, 1 P2P, 2 staged) */
static int classify(const Oracle* o, int a, int b) {
    if (a == b) return 0;
    return o->p2p[(size_t)a * o->devices + b] ? 1 : 2;
}
/* proj/src/topology.cpp:96-111 */
static double f_cost(const Oracle* o, int cand, const int* owners, int n) {
    double sum = 0.0;
    for (int k = 0; k < n; ++k) {
        const int cls = classify(o, cand, owners[k]);
        sum += cls == 0 ? 0.0
               : cls == 1 ? o->weight_p2p * (double)o->face_xfer
                          : o->weight_staged * (double)o->face_xfer;
    }
    return sum;
}
/* proj/src/assign.cpp:8-38 */
static int assign_device(Oracle* o, const int* owners, int n) {
    unsigned long long lo = o->per_dev[0];
    for (int d = 1; d < o->devices; ++d)
        if (o->per_dev[d] < lo) lo = o->per_dev[d];
    int chosen = -1;
    double best = 0.0;
    for (int d = 0; d < o->devices; ++d) {
        if (o->per_dev[d] != lo) continue;
        if (chosen < 0) {
            chosen = d;
            if (o->policy == PLBM_POLICY_SIMPLE) break;
            best = f_cost(o, d, owners, n);
        } else {
            const double c = f_cost(o, d, owners, n);
            if (c < best) { best = c; chosen = d; }
        }
    }
    ++o->per_dev[chosen];
    return chosen;
}
/* proj/src/engine.cpp:30-41 */
static void assign_owner(Oracle* o, Tile* t) {
    int owners[6], n = 0;
    for (int f = 0; f < 6; ++f) {
        const Tile* nb = neighbor(o, t, f);
        if (nb && nb->owner >= 0 && nb != t) owners[n++] = nb->owner;
    }
    const int dev = assign_device(o, owners, n);
    t->owner = dev;
    o->log[t->log_index].owner = dev;
}
/* proj/src/topology.cpp:113-117 */
static void record_exchange(Oracle* o, int a, int b) {
    o->bytes[classify(o, a, b)] += o->face_xfer;
}

/* proj/src/scenario.cpp:177-183 */
static int seed_contains(const plbm_seed_desc* s, double x, double y, double z) {
    if (s->shape == PLBM_SEED_BOX)
        return x >= s->box_min[0] && x < s->box_max[0] && y >= s->box_min[1] &&
               y < s->box_max[1] && z >= s->box_min[2] && z < s->box_max[2];
    const double dx = x - s->center[0], dy = y - s->center[1], dz = z - s->center[2];
    return dx * dx + dy * dy + dz * dz <= s->radius * s->radius;
}

/* ---------------------------------------------------------------- L3 */

static void set_error(Oracle* o, const Tile* t, long it, const char* phase, const char* msg) {
    if (o->err) return;
    o->err = 1;
    memcpy(o->err_tile, t->c, sizeof o->err_tile);
    o->err_it = it;
    snprintf(o->err_phase, sizeof o->err_phase, "%s", phase);
    snprintf(o->err_msg, sizeof o->err_msg, "iteration %ld, tile (%d,%d,%d), phase %s: %s",
             it, t->c[0], t->c[1], t->c[2], phase, msg);
}

#define FOR_TILES(o, t)                                           \
    for (size_t _k = 0, _n = (size_t)(o)->grid[0] * (o)->grid[1] * (o)->grid[2]; _k < _n; ++_k) \
        for (Tile* t = (o)->tiles[_k]; t; t = NULL)

/* proj/src/engine.cpp:221-264 (P1) */
static void phase1(Oracle* o) {
    const long it = o->iteration + 1;
    const size_t gc = o->gcells;
    FOR_TILES(o, t) {
        if (o->err) return;
        for (int c = 0; c < o->C; ++c) {
            const plbm_component_desc* par = &o->comp[c];
            memcpy(t->pux + c * gc, t->ux + c * gc, gc * sizeof(double));
            memcpy(t->puy + c * gc, t->uy + c * gc, gc * sizeof(double));
            memcpy(t->puz + c * gc, t->uz + c * gc, gc * sizeof(double));
            const double* f = t->f[t->cur] + (size_t)c * Q * gc;
            for (int pass = 0; pass < 2; ++pass) {
                const int* cells = pass ? t->icells : t->bcells;
                const int n = pass ? t->ni : t->nb;
                for (int k = 0; k < n; ++k) {
                    const size_t cell = (size_t)cells[k];
                    double rho = 0.0;
                    for (int i = 0; i < Q; ++i) {
                        const double v = f[(size_t)i * gc + cell];
                        rho += v;
                        if (v < 0.0) ++o->neg;
                    }
                    if (!isfinite(rho)) { set_error(o, t, it, "P1", "NaN in density"); return; }
                    double press;
                    if (pr_pressure(rho, par, &press)) {
                        set_error(o, t, it, "P1", "pr_pressure: b*rho >= 1 (EOS pole)");
                        return;
                    }
                    t->rho[c * gc + cell] = rho;
                    t->psi[c * gc + cell] = pseudo_potential(rho, press, par->g_self, &o->clamps);
                }
            }
        }
    }
}

/* proj/src/engine.cpp:274-296 — destination slab of one ghost pass. */
typedef struct { int lo[3], hi[3], src_shift; } Slab;
static Slab make_slab(const Oracle* o, int axis, int dir) {
    Slab s;
    const int g = o->g;
    for (int b = 0; b < 3; ++b) {
        if (b == axis) {
            const int ghost = dir < 0 ? 0 : g - 1;
            s.lo[b] = ghost; s.hi[b] = ghost + 1;
        } else if (b < axis) {
            s.lo[b] = 0; s.hi[b] = g;
        } else {
            s.lo[b] = 1; s.hi[b] = g - 1;
        }
    }
    s.src_shift = dir < 0 ? g - 2 : -(g - 2);
    return s;
}

/* proj/src/engine.cpp:298-391 — P2 (psi) and P4a (populations) passes. */
static void ghost_pass(Oracle* o, int axis, int populations) {
    const size_t gc = o->gcells;
    const long stride[3] = {1, o->g, (long)o->g * o->g};
    FOR_TILES(o, t) {
        for (int dir = -1; dir <= 1; dir += 2) {
            const int face = 2 * axis + (dir < 0 ? 0 : 1);
            Tile* nb = neighbor(o, t, face);
            const Slab sl = make_slab(o, axis, dir);
            const long src_off = sl.src_shift * stride[axis];
            for (int c = 0; c < o->C; ++c) {
                const int nplanes = populations ? Q : 1;
                for (int i = 0; i < nplanes; ++i) {
                    double* dst = populations ? t->f[t->cur] + ((size_t)c * Q + i) * gc
                                              : t->psi + (size_t)c * gc;
                    const double* src = NULL;
                    if (nb) src = populations ? nb->f[nb->cur] + ((size_t)c * Q + i) * gc
                                              : nb->psi + (size_t)c * gc;
                    for (int z = sl.lo[2]; z < sl.hi[2]; ++z)
                        for (int y = sl.lo[1]; y < sl.hi[1]; ++y)
                            for (int x = sl.lo[0]; x < sl.hi[0]; ++x) {
                                const long cell = x + stride[1] * y + stride[2] * z;
                                if (nb) dst[cell] = src[cell + src_off];
                                else if (populations) dst[cell] = o->amb_feq[c][i];
                                else dst[cell] = t->solid[cell] ? 0.0 : o->amb_psi[c];
                            }
                }
            }
            if (nb) record_exchange(o, t->owner, nb->owner);
        }
    }
}

/* proj/src/engine.cpp:407-479 */
static void collide_cells(Oracle* o, Tile* t, const int* cells, int n) {
    const size_t gc = o->gcells;
    const long stride[3] = {1, o->g, (long)o->g * o->g};
    for (int c = 0; c < o->C; ++c) {
        const plbm_component_desc* par = &o->comp[c];
        double* f = t->f[t->cur] + (size_t)c * Q * gc;
        const int has_gravity = par->gravity[0] != 0.0 || par->gravity[1] != 0.0 ||
                                par->gravity[2] != 0.0;
        const double omega = 1.0 / par->tau;
        for (int k = 0; k < n; ++k) {
            const size_t cell = (size_t)cells[k];
            const double rho = t->rho[c * gc + cell];
            const double u[3] = {t->ux[c * gc + cell], t->uy[c * gc + cell], t->uz[c * gc + cell]};
            double F[3] = {0, 0, 0};
            if (has_gravity) {
                F[0] = rho * par->gravity[0];
                F[1] = rho * par->gravity[1];
                F[2] = rho * par->gravity[2];
            }
            double Fi[3];
            intra_force(t->psi + c * gc, (long)cell, stride, par, Fi);
            F[0] += Fi[0]; F[1] += Fi[1]; F[2] += Fi[2];
            for (int c2 = 0; c2 < o->C; ++c2) {
                if (c2 == c) continue;
                const double gx = o->coupling[c * o->C + c2];
                if (gx == 0.0) continue;
                double Fx[3];
                inter_force(t->psi[c * gc + cell], t->psi + c2 * gc, (long)cell, stride, gx, Fx);
                F[0] += Fx[0]; F[1] += Fx[1]; F[2] += Fx[2];
            }
            double eq0[Q];
            equilibrium(rho, u, eq0);
            if (F[0] == 0.0 && F[1] == 0.0 && F[2] == 0.0) {
                for (int i = 0; i < Q; ++i) {
                    const size_t kk = (size_t)i * gc + cell;
                    f[kk] += omega * (eq0[i] - f[kk]);
                }
            } else if (rho <= 0.0) {
                ++o->zero_rho;
                for (int i = 0; i < Q; ++i) {
                    const size_t kk = (size_t)i * gc + cell;
                    f[kk] += omega * (eq0[i] - f[kk]);
                }
            } else {
                const double us[3] = {u[0] + F[0] / rho, u[1] + F[1] / rho, u[2] + F[2] / rho};
                double eq1[Q];
                equilibrium(rho, us, eq1);
                for (int i = 0; i < Q; ++i) {
                    const size_t kk = (size_t)i * gc + cell;
                    f[kk] += omega * (eq0[i] - f[kk]) + eq1[i] - eq0[i];
                }
            }
        }
    }
}

/* proj/src/tilemap.cpp:182-218 */
static int evaluate_criterion(Oracle* o, const Tile* t, int faces[6]) {
    int n_out = 0;
    const double s2 = o->threshold * o->threshold;
    const int E = o->E;
    const size_t gc = o->gcells;
    for (int fi = 0; fi < 6; ++fi) {
        if (neighbor(o, t, fi) != NULL) continue;
        const int axis = fi / 2;
        const int fixed = (fi % 2) ? E - 1 : 0;
        int lo[3] = {0, 0, 0}, hi[3] = {E, E, E};
        lo[axis] = fixed; hi[axis] = fixed + 1;
        int fired = 0;
        for (int c = 0; c < o->C && !fired; ++c)
            for (int lz = lo[2]; lz < hi[2] && !fired; ++lz)
                for (int ly = lo[1]; ly < hi[1] && !fired; ++ly)
                    for (int lx = lo[0]; lx < hi[0]; ++lx) {
                        const size_t cell = gidx(o, lx, ly, lz);
                        if (t->solid[cell]) continue;
                        const size_t k = c * gc + cell;
                        const double dx = t->ux[k] - t->pux[k];
                        const double dy = t->uy[k] - t->puy[k];
                        const double dz = t->uz[k] - t->puz[k];
                        if (dx * dx + dy * dy + dz * dz > s2) { fired = 1; break; }
                    }
        if (fired) faces[n_out++] = fi;
    }
    return n_out;
}

/* proj/src/engine.cpp:482-527 (P4 stream + P5 moments/criterion) */
static void phase5(Oracle* o, Trigger** trig, size_t* n_trig, size_t* cap_trig) {
    const long it = o->iteration + 1;
    const size_t gc = o->gcells;
    FOR_TILES(o, t) {
        for (int c = 0; c < o->C; ++c) {
            const double* f = t->f[t->cur] + (size_t)c * Q * gc;
            for (int pass = 0; pass < 2; ++pass) {
                const int* cells = pass ? t->icells : t->bcells;
                const int n = pass ? t->ni : t->nb;
                for (int k = 0; k < n; ++k) {
                    const size_t cell = (size_t)cells[k];
                    double fi[Q], rho, u[3];
                    for (int i = 0; i < Q; ++i) fi[i] = f[(size_t)i * gc + cell];
                    moments(fi, &rho, u);
                    if (!isfinite(rho) || !isfinite(u[0]) || !isfinite(u[1]) || !isfinite(u[2])) {
                        set_error(o, t, it, "P5", "NaN in moments");
                        return;
                    }
                    t->rho[c * gc + cell] = rho;
                    t->ux[c * gc + cell] = u[0];
                    t->uy[c * gc + cell] = u[1];
                    t->uz[c * gc + cell] = u[2];
                }
            }
        }
        if (o->mode == PLBM_MODE_PROGRESSIVE) {
            int faces[6];
            const int nf = evaluate_criterion(o, t, faces);
            for (int k = 0; k < nf; ++k) {
                if (*n_trig == *cap_trig) {
                    *cap_trig = *cap_trig ? 2 * *cap_trig : 64;
                    *trig = (Trigger*)realloc(*trig, *cap_trig * sizeof(Trigger));
                }
                Trigger tr = {{t->c[0], t->c[1], t->c[2]}, faces[k]};
                (*trig)[(*n_trig)++] = tr;
            }
        }
    }
}

typedef struct { int target[3], source[3], face, in_bounds; } Resolved;
static int cmp3(const int* a, const int* b) {
    for (int k = 0; k < 3; ++k)
        if (a[k] != b[k]) return a[k] < b[k] ? -1 : 1;
    return 0;
}
/* proj/src/tilemap.cpp:242-247 ordering */
static int cmp_resolved(const void* pa, const void* pb) {
    const Resolved* a = (const Resolved*)pa;
    const Resolved* b = (const Resolved*)pb;
    if (a->in_bounds != b->in_bounds) return a->in_bounds > b->in_bounds ? -1 : 1;
    int c = cmp3(a->target, b->target);
    if (c) return c;
    c = cmp3(a->source, b->source);
    if (c) return c;
    return a->face - b->face;
}
static int cmp_tile_ptr(const void* pa, const void* pb) {
    return cmp3((*(Tile* const*)pa)->c, (*(Tile* const*)pb)->c);
}

/* proj/src/tilemap.cpp:220-266 + engine.cpp:554-560 */
static void expand_and_assign(Oracle* o, Trigger* trig, size_t n, long iteration) {
    Resolved* rs = (Resolved*)malloc((n ? n : 1) * sizeof(Resolved));
    for (size_t k = 0; k < n; ++k) {
        int tgt[3] = {0, 0, 0};
        const int ok = neighbor_coords(o, trig[k].src, trig[k].face, tgt);
        Resolved r;
        memcpy(r.target, ok ? tgt : (int[3]){0, 0, 0}, sizeof r.target);
        memcpy(r.source, trig[k].src, sizeof r.source);
        r.face = trig[k].face;
        r.in_bounds = ok;
        rs[k] = r;
    }
    qsort(rs, n, sizeof(Resolved), cmp_resolved);
    Tile** created = (Tile**)malloc((n ? n : 1) * sizeof(Tile*));
    size_t n_created = 0;
    const int* last = NULL;
    for (size_t k = 0; k < n; ++k) {
        if (!rs[k].in_bounds) { ++o->suppressed; continue; }
        if (last && cmp3(rs[k].target, last) == 0) continue;
        last = rs[k].target;
        if (at(o, rs[k].target[0], rs[k].target[1], rs[k].target[2])) continue;
        created[n_created++] = create_tile(o, rs[k].target, iteration, rs[k].face);
    }
    qsort(created, n_created, sizeof(Tile*), cmp_tile_ptr);
    for (size_t k = 0; k < n_created; ++k) assign_owner(o, created[k]);
    free(created);
    free(rs);
}

/* proj/src/engine.cpp:537-563 — one iteration. */
static int oracle_step(Oracle* o) {
    const unsigned long long updates = o->active_cells;
    phase1(o);
    if (o->err) return 1;
    for (int a = 0; a < 3; ++a) ghost_pass(o, a, 0);
    FOR_TILES(o, t) {
        collide_cells(o, t, t->bcells, t->nb);
        collide_cells(o, t, t->icells, t->ni);
    }
    for (int a = 0; a < 3; ++a) ghost_pass(o, a, 1);
    FOR_TILES(o, t) {
        for (int c = 0; c < o->C; ++c)
            stream_pull(t->f[t->cur] + (size_t)c * Q * o->gcells,
                        t->f[1 - t->cur] + (size_t)c * Q * o->gcells, t->solid, o->g);
        t->cur = 1 - t->cur;
    }
    Trigger* trig = NULL;
    size_t n_trig = 0, cap_trig = 0;
    phase5(o, &trig, &n_trig, &cap_trig);
    if (o->err) { free(trig); return 1; }
    if (o->mode == PLBM_MODE_PROGRESSIVE) expand_and_assign(o, trig, n_trig, o->iteration + 1);
    free(trig);
    ++o->iteration;
    o->cell_updates += updates;
    return 0;
}

/* ---------------------------------------------------------------- API */

static void set_api_err(plbm_error* e, int code, const char* msg) {
    if (!e) return;
    memset(e, 0, sizeof *e);
    e->code = code;
    snprintf(e->message, sizeof e->message, "%s", msg);
}

/* proj/src/engine.cpp:91-161 (make_state) — validation is the caller's. */
void* plbm_oracle_create(const plbm_scenario_desc* d, int workers, plbm_error* err) {
    (void)workers;
    set_api_err(err, 0, "");
    init_opp();
    if (d->n_components < 1 || d->n_components > PLBM_MAX_COMP ||
        d->n_seeds < 0 || d->n_seeds > PLBM_MAX_SEEDS || d->tile_extent < 4) {
        set_api_err(err, 2, "oracle: unsupported scenario shape");
        return NULL;
    }
    for (int a = 0; a < 3; ++a)
        if (d->domain[a] % d->tile_extent != 0) {
            set_api_err(err, 2, "oracle: domain not divisible by tile_extent");
            return NULL;
        }
    if (d->mode == PLBM_MODE_PROGRESSIVE && d->n_seeds == 0) {
        set_api_err(err, 2, "config: progressive mode requires at least one seed region");
        return NULL;
    }
    Oracle* o = (Oracle*)calloc(1, sizeof(Oracle));
    for (int a = 0; a < 3; ++a) {
        o->dom[a] = d->domain[a];
        o->periodic[a] = d->periodic[a];
        o->grid[a] = d->domain[a] / d->tile_extent;
    }
    o->E = d->tile_extent;
    o->g = o->E + 2;
    o->gcells = (size_t)o->g * o->g * o->g;
    o->C = d->n_components;
    o->mode = d->mode;
    o->threshold = d->threshold;
    o->devices = d->devices;
    o->policy = d->policy;
    o->weight_p2p = d->weight_p2p;
    o->weight_staged = d->weight_staged;
    memcpy(o->comp, d->components, sizeof(plbm_component_desc) * (size_t)o->C);
    if (d->coupling) memcpy(o->coupling, d->coupling, sizeof(double) * (size_t)(o->C * o->C));
    o->n_seeds = d->n_seeds;
    if (d->n_seeds) memcpy(o->seeds, d->seeds, sizeof(plbm_seed_desc) * (size_t)d->n_seeds);
    const size_t ncells = (size_t)o->dom[0] * o->dom[1] * o->dom[2];
    if (d->geometry) {
        o->geom = (unsigned char*)malloc(ncells);
        memcpy(o->geom, d->geometry, ncells);
    }
    o->p2p = (unsigned char*)malloc((size_t)o->devices * o->devices);
    for (int k = 0; k < o->devices * o->devices; ++k) o->p2p[k] = d->p2p ? d->p2p[k] : 1;
    o->per_dev = (unsigned long long*)calloc((size_t)o->devices, sizeof(unsigned long long));
    /* proj/src/tilemap.cpp:13-28 */
    for (int c = 0; c < o->C; ++c) {
        double press = 0.0;
        o->amb_rho[c] = o->comp[c].rho_ambient;
        pr_pressure(o->comp[c].rho_ambient, &o->comp[c], &press);
        o->amb_psi[c] = pseudo_potential(o->comp[c].rho_ambient, press, o->comp[c].g_self, NULL);
        const double u0[3] = {0, 0, 0};
        equilibrium(o->comp[c].rho_ambient, u0, o->amb_feq[c]);
    }
    /* proj/src/engine.cpp:128-132; proj/src/topology.cpp:85-89 */
    o->face_xfer = (unsigned long long)o->E * o->E * (unsigned long long)o->C * (5 + 1) * 8;
    const size_t ntile = (size_t)o->grid[0] * o->grid[1] * o->grid[2];
    o->tiles = (Tile**)calloc(ntile, sizeof(Tile*));
    /* initial tile set, proj/src/engine.cpp:135-158 */
    unsigned char* initial = (unsigned char*)calloc(ntile, 1);
    if (o->mode == PLBM_MODE_STATIC) {
        memset(initial, 1, ntile);
    } else {
        for (int s = 0; s < o->n_seeds; ++s)
            for (int z = 0; z < o->dom[2]; ++z)
                for (int y = 0; y < o->dom[1]; ++y)
                    for (int x = 0; x < o->dom[0]; ++x)
                        if (seed_contains(&o->seeds[s], x + 0.5, y + 0.5, z + 0.5))
                            initial[lin(o, x / o->E, y / o->E, z / o->E)] = 1;
    }
    for (size_t k = 0; k < ntile; ++k) {
        if (!initial[k]) continue;
        const int c[3] = {(int)(k / ((size_t)o->grid[1] * o->grid[2])),
                          (int)((k / o->grid[2]) % o->grid[1]), (int)(k % o->grid[2])};
        Tile* t = create_tile(o, c, 0, -1);
        assign_owner(o, t);
    }
    free(initial);
    /* apply_seeds, proj/src/engine.cpp:43-76 */
    const size_t gc = o->gcells;
    for (int s = 0; s < o->n_seeds; ++s) {
        const plbm_seed_desc* sd = &o->seeds[s];
        double feq[Q];
        const double u[3] = {sd->velocity[0], sd->velocity[1], sd->velocity[2]};
        equilibrium(sd->rho, u, feq);
        const int c = sd->component;
        FOR_TILES(o, t) {
            for (int lz = 0; lz < o->E; ++lz)
                for (int ly = 0; ly < o->E; ++ly)
                    for (int lx = 0; lx < o->E; ++lx) {
                        const size_t cell = gidx(o, lx, ly, lz);
                        if (t->solid[cell]) continue;
                        if (!seed_contains(sd, t->c[0] * o->E + lx + 0.5, t->c[1] * o->E + ly + 0.5,
                                           t->c[2] * o->E + lz + 0.5))
                            continue;
                        for (int i = 0; i < Q; ++i) {
                            t->f[0][((size_t)c * Q + i) * gc + cell] = feq[i];
                            t->f[1][((size_t)c * Q + i) * gc + cell] = feq[i];
                        }
                        t->rho[c * gc + cell] = sd->rho;
                        t->ux[c * gc + cell] = u[0];
                        t->uy[c * gc + cell] = u[1];
                        t->uz[c * gc + cell] = u[2];
                    }
        }
    }
    return o;
}

int plbm_oracle_step(void* h, int n, plbm_error* err) {
    Oracle* o = (Oracle*)h;
    set_api_err(err, 0, "");
    for (int k = 0; k < n; ++k) {
        if (oracle_step(o)) {
            set_api_err(err, 1, o->err_msg);
            if (err) {
                memcpy(err->tile, o->err_tile, sizeof err->tile);
                err->iteration = o->err_it;
                snprintf(err->phase, sizeof err->phase, "%s", o->err_phase);
            }
            o->err = 0;
            return 1;
        }
    }
    return 0;
}

void plbm_oracle_counters(void* h, plbm_counters* out) {
    const Oracle* o = (const Oracle*)h;
    memset(out, 0, sizeof *out);
    out->iteration = o->iteration;
    out->cell_updates = o->cell_updates;
    out->negative_populations = o->neg;
    out->psi_clamps = o->clamps;
    out->zero_rho_forcings = o->zero_rho;
    out->suppressed_expansions = o->suppressed;
    for (int k = 0; k < 3; ++k) out->bytes[k] = o->bytes[k];
    out->tiles = (uint64_t)o->n_tiles;
    out->active_cells = o->active_cells;
    /* proj/src/tile.cpp:7-13 */
    out->bytes_resident = (uint64_t)o->n_tiles * o->gcells *
                          ((uint64_t)o->C * (2 * Q + 8) * 8 + 1);
}

int plbm_oracle_tiles(void* h, int32_t* coords, int32_t* owners, int64_t* births, int max) {
    const Oracle* o = (const Oracle*)h;
    int k = 0;
    FOR_TILES(o, t) {
        if (k < max) {
            if (coords) { coords[3 * k] = t->c[0]; coords[3 * k + 1] = t->c[1]; coords[3 * k + 2] = t->c[2]; }
            if (owners) owners[k] = t->owner;
            if (births) births[k] = t->birth;
        }
        ++k;
    }
    return k;
}

int plbm_oracle_read_tile(void* h, const int32_t* coords, int comp, int field, double* out) {
    const Oracle* o = (const Oracle*)h;
    if (coords[0] < 0 || coords[0] >= o->grid[0] || coords[1] < 0 || coords[1] >= o->grid[1] ||
        coords[2] < 0 || coords[2] >= o->grid[2])
        return -1;
    const Tile* t = at(o, coords[0], coords[1], coords[2]);
    if (!t) return -1;
    if (comp < 0 || comp >= o->C) return -2;
    const int E = o->E;
    const size_t gc = o->gcells, n = (size_t)E * E * E;
    const double* src;
    switch (field) {
    case PLBM_FIELD_F: src = NULL; break;
    case PLBM_FIELD_RHO: src = t->rho; break;
    case PLBM_FIELD_UX: src = t->ux; break;
    case PLBM_FIELD_UY: src = t->uy; break;
    case PLBM_FIELD_UZ: src = t->uz; break;
    case PLBM_FIELD_PUX: src = t->pux; break;
    case PLBM_FIELD_PUY: src = t->puy; break;
    case PLBM_FIELD_PUZ: src = t->puz; break;
    case PLBM_FIELD_PSI: src = t->psi; break;
    default: return -3;
    }
    const int planes = field == PLBM_FIELD_F ? Q : 1;
    for (int i = 0; i < planes; ++i) {
        const double* p = field == PLBM_FIELD_F
                              ? t->f[t->cur] + ((size_t)comp * Q + i) * gc
                              : src + (size_t)comp * gc;
        for (int z = 0; z < E; ++z)
            for (int y = 0; y < E; ++y)
                for (int x = 0; x < E; ++x)
                    out[i * n + (size_t)x + (size_t)E * ((size_t)y + (size_t)E * z)] =
                        p[gidx(o, x, y, z)];
    }
    return 0;
}

int plbm_oracle_creation_log(void* h, plbm_creation_event* out, int max) {
    const Oracle* o = (const Oracle*)h;
    for (size_t k = 0; k < o->n_log && (int)k < max; ++k) {
        out[k].iteration = o->log[k].iteration;
        memcpy(out[k].coords, o->log[k].c, sizeof out[k].coords);
        out[k].trigger = o->log[k].trigger;
        out[k].owner = o->log[k].owner;
        out[k].pad = 0;
    }
    return (int)o->n_log;
}

int plbm_oracle_poke_f(void* h, const int32_t* coords, int comp, int i, const int32_t* local, double v) {
    Oracle* o = (Oracle*)h;
    Tile* t = at(o, coords[0], coords[1], coords[2]);
    if (!t) return -1;
    t->f[t->cur][((size_t)comp * Q + i) * o->gcells + gidx(o, local[0], local[1], local[2])] = v;
    return 0;
}

void plbm_oracle_destroy(void* h) {
    Oracle* o = (Oracle*)h;
    if (!o) return;
    const size_t ntile = (size_t)o->grid[0] * o->grid[1] * o->grid[2];
    for (size_t k = 0; k < ntile; ++k) free_tile(o->tiles[k]);
    free(o->tiles); free(o->log); free(o->geom); free(o->p2p); free(o->per_dev);
    free(o);
}

/* ---------------------------------------------------------------- KATs
 * Single-function entry points so the restatement can be checked against
 * the reference's own known-answer unit tests (tests/test_golden.py). */
double plbm_oracle_kat_pr_pressure(double rho, const plbm_component_desc* p, int* pole) {
    double out = 0.0;
    *pole = pr_pressure(rho, p, &out);
    return out;
}
double plbm_oracle_kat_psi(double rho, double press, double g_self, int* clamped) {
    unsigned long long c = 0;
    const double v = pseudo_potential(rho, press, g_self, &c);
    *clamped = (int)c;
    return v;
}
void plbm_oracle_kat_equilibrium(double rho, const double* u, double* out) {
    init_opp();
    equilibrium(rho, u, out);
}
void plbm_oracle_kat_moments(const double* f, double* rho, double* u) { moments(f, rho, u); }
void plbm_oracle_kat_intra_force(const double* psi, long cell, const long* stride,
                                 const plbm_component_desc* p, double* F) {
    intra_force(psi, cell, stride, p, F);
}
void plbm_oracle_kat_inter_force(double psi_self, const double* psi_other, long cell,
                                 const long* stride, double g, double* F) {
    inter_force(psi_self, psi_other, cell, stride, g, F);
}
void plbm_oracle_kat_stencil(int* e, double* w, int* opp) {
    init_opp();
    for (int i = 0; i < Q; ++i) {
        for (int a = 0; a < 3; ++a) e[3 * i + a] = E3[i][a];
        w[i] = W3[i];
        opp[i] = OPP[i];
    }
}
