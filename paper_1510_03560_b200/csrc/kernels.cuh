// kernels.cuh — the B200 step-loop kernels (sm_100a, FP64, no tensor cores).
//
// Storage (HBM block pool, SoA), addressed through per-slot pointer tables so
// that a slot may live on this GPU or on a peer GPU (read over NVLink):
//   slot_f[b][s]  : -> [comp][19][E^3] doubles of slot s in buffer b (A-B).
//                   The stored state is the POST-COLLISION population of the
//                   last step (f_post^(k)); the reference's post-stream f_read
//                   is produced on the fly by pulling (stream fused into the
//                   next step's load).
//   slot_pf[p][s] : -> [comp][6][E^2] face-layer psi of slot s for the step of
//                   parity p (written by k_face at the end of the previous step,
//                   read by neighbours in k_main; double-buffered so a peer can
//                   still read step k's faces while this GPU writes step k+1's).
//   AMB slot      : one extra slot (global id = capacity) holding feq_amb in both
//                   buffers and psi_amb on its faces; every route to an absent
//                   tile points at it, so frontier pulls need no branch.
//   route[r]      : [slot][18] source slot for the 6 face and 12 edge ghost
//                   classes, resolved with the reference's ghost-routing rule
//                   (hop along the higher axis first; proj/src/engine.cpp:266-296).
//                   ROUTE_PULL = map of the previous step (P4 of the last step ran
//                   on it), ROUTE_PSI = map of this step (P2 runs on it).
//   u_face        : [local][comp][6][3][E^2] velocity used by the last collision
//                   on frontier faces (u_prev of the activation criterion).
//
// Per step k:
//   k_main* : pull f_in^(k) from f_post^(k-1) (or generate it for seeded /
//             newborn tiles), rho/psi planes in shared memory marching in z,
//             Shan-Chen forces, BGK + velocity-shift forcing, store f_post^(k).
//             = reference P1 + P2 + P3 + P4 + (P5 moments of the previous step).
//   k_face  : moments of f_in^(k+1) on the 6 face layers: psi faces for step
//             k+1 and the activation criterion of step k (P5 + evaluate_criterion).
#pragma once

#include "lattice.cuh"

namespace plbm {

enum TileMode : uint8_t { MODE_PULL = 0, MODE_GEN_SEEDED = 1, MODE_GEN_AMBIENT = 2 };
enum { ROUTE_PULL = 0, ROUTE_PSI = 1, ROUTE_W = 2 };
// Population storage.  A-B (AA_OFF): two buffers, step k pulls f_post^(k-1)
// from one and stores f_post^(k) into the other.  A-A (SURVEY §8(f)3,
// PAPER.md:85): ONE buffer updated in place, the step kinds alternating
//   AA_LOCAL (odd steps):  cell x reads (x, i) for every i and stores
//                          f_post(x)[i] at (x, opp i);
//   AA_NEIGH (even steps): cell x reads f_post(x - e_i)[i] at (x - e_i, opp i)
//                          (bounce-back: f_post(x)[opp i] at (x, i)) and stores
//                          f_post(x)[i] at (x + e_i, i), or at (x, opp i) when
//                          x + e_i is solid.
// Every location (cell, dir) is read and written by exactly one cell in a
// step, so no step needs a second buffer.  Frontier rules are the A-B ones:
// a source in an absent tile (ROUTE_PULL -> ambient) reads feq_amb[i]; a store
// into an absent geometric neighbour (ROUTE_W -> ambient) is dropped (nobody
// reads it: a tile born later starts from feq_amb, GEN_AMBIENT).
enum { AA_OFF = 0, AA_LOCAL = 1, AA_NEIGH = 2 };
__host__ __device__ inline int aa_kind(int aa, long iter) {
    return aa ? ((iter & 1) ? AA_LOCAL : AA_NEIGH) : AA_OFF;
}
enum { ERR_NONE = 0, ERR_P1_NAN = 1, ERR_P1_POLE = 2, ERR_P5_NAN = 3, ERR_PEER_TIMEOUT = 4 };
// "no error" value of the error key (atomicMin; also an int64 MAX so a
// signed MIN reduction across ranks keeps the earliest key)
constexpr unsigned long long ERR_NONE_KEY = 0x7fffffffffffffffull;
enum { CNT_NEG = 0, CNT_CLAMP = 1, CNT_ZERO_RHO = 2, CNT_SUPP = 3, CNT_N = 4 };

constexpr int MAX_COMP = 4;
constexpr int MAX_SEEDS = 64;

struct SeedConst {
    int shape, comp;
    double lo[3], hi[3], center[3], r2;
    double rho, u[3];
    double feq[Q];
};

struct Params {
    int C;
    int n_seeds;
    int grid[3];
    int amb_slot;
    int progressive;
    double s2;  // threshold^2 (tilemap.cpp:185)
    int mid_sp; // rows between the mid-face boundaries (E / finest clusters per tile; 0: none)
    CompConst comp[MAX_COMP];
    double coupling[MAX_COMP * MAX_COMP];
    SeedConst seeds[MAX_SEEDS];
};

struct Dev {
    double* const* slot_f[2];   // [slot] -> f block in buffer b (local or peer)
    double* const* slot_pf[2];  // [slot] -> psi faces for step parity p
    const int* route[3];        // [slot][18]: ROUTE_PULL, ROUTE_PSI, ROUTE_W (geometric, A-A stores)
    int aa;                     // 1: A-A in-place storage (slot_f[0] == slot_f[1])
    const int* lidx;            // [slot] -> local index (u_face / capture), -1 remote
    const uint32_t* solid;      // [slot][solid_words]
    const uint8_t* has_solid;   // [slot]
    const uint8_t* mode;        // [slot]
    const int* coords;          // [slot][3]
    double* u_face;             // [local][C][6][3][E2]
    uint8_t* trig;              // [slot]
    double* capture;            // [local][C][4][E3] or nullptr
    unsigned long long* cnt;    // CNT_N
    unsigned long long* err;    // packed (iter, tile_lin, code), atomicMin
    int solid_words;
    // fused face pass (single rank): the cluster that completes the last of a
    // tile's 19 dependencies (itself + geometric neighbours) runs its face pass
    int* dep_cnt;               // [slot] completions this step (self-resetting)
    const int* dep_need;        // [slot] 1 + active geometric neighbours
    const int* geo;             // [slot][18] active geometric neighbour or -1
    int face_flags;             // FACE_* bits
    int xcol_ok;                // the last fused kernel wrote the xcol side buffers
    int mid_faces;              // the face pass also writes psi of the rows on both sides of
                                // every y = b * P.mid_sp boundary (faces 6.., the boundary rows
                                // of clusters covering part of a tile), after the 6 faces
    const int* halt;            // speculative queue: a step kernel finding *halt != 0 does nothing
    const struct Poke* pokes;   // test hook (plbm_gpu_poke_f): overrides of f_in for the next step
    int npoke;
    const int* nactive;         // device-side expansion: tiles beyond *nactive in the launch are idle
    unsigned long long* probe;  // measurement: per-CTA {smid, start, end} globaltimer (or nullptr)
    int tile_base;              // this launch's tiles start at active[tile_base] (co-scheduled split)
    uint8_t* suspect;           // [slot] P5 screen: a stored f_post value left [2^-400, 2^400)
    int screen_all;             // the ambient populations fail the screen: k_p5 checks every tile
    unsigned* susp_any;         // [2] by step parity: some tile was marked (nullptr: multi-rank)
    int neg_exact;              // always count negative populations with FP compares (see k_main_pc)
    // [slot] 1 = the tile has no fluid cell.  Nothing ever reads such a tile:
    // a fluid cell next to a solid one bounces back (its own populations), a
    // solid ghost's psi is 0 from the reader's own solid mask, and a reader
    // without solids (the only one using xcol) cannot border it.  Its
    // fused-kernel and face-pass CTAs exit at once (state, counters and
    // read-back are unaffected: it has no fluid cell to update or report).
    const uint8_t* no_fluid;
};

__device__ __forceinline__ unsigned long long global_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ unsigned smid() {
    unsigned s;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(s));
    return s;
}

struct Poke {
    int slot, comp, i, cell;
    double v;
};

// plbm_gpu_poke_f: the reference overwrites f_read between steps
// (proj/tests/test_engine.cpp:284-310); here the override is applied to the
// pulled f_in of the next step's psi pass.  f stays in registers (the
// direction index is matched against the unrolled loop).
template <int E>
__device__ __forceinline__ void apply_pokes(const Dev& d, int slot, int c, int x, int y, int z, double* f) {
    if (d.npoke == 0) return;
    const int cell = (z * E + y) * E + x;
    for (int k = 0; k < d.npoke; ++k) {
        const Poke p = d.pokes[k];
        if (p.slot != slot || p.comp != c || p.cell != cell) continue;
#pragma unroll
        for (int i = 0; i < Q; ++i)
            if (i == p.i) f[i] = p.v;
    }
}

// Speculatively queued steps (Engine::step, single rank, progressive): every
// step kernel first checks the sticky halt flag that k_check sets when the
// previous step's triggers need the host (a birth) or an error occurred.
__device__ __forceinline__ bool halted(const Dev& d) {
    return d.halt && *(volatile const int*)d.halt != 0;
}
enum { FACE_CRITERION = 1, FACE_NAN = 2, FACE_FUSED = 4 };

static __constant__ Params P;  // one copy per translation unit (dispatch.cuh)

// 18 ghost classes: 0..5 faces (-x,+x,-y,+y,-z,+z), 6..17 edges.
__host__ __device__ inline int edge_class(int a, int b, int da, int db) {
    const int pair = (a == 0) ? (b == 1 ? 0 : 1) : 2;
    return 6 + 4 * pair + (da > 0 ? 1 : 0) + (db > 0 ? 2 : 0);
}
// out pattern (ox,oy,oz) in {-1,0,1}^3 with 1 or 2 non-zeros -> class
__host__ __device__ inline int ghost_class(int ox, int oy, int oz) {
    const int n = (ox != 0) + (oy != 0) + (oz != 0);
    if (n == 1) {
        if (ox) return ox > 0 ? 1 : 0;
        if (oy) return oy > 0 ? 3 : 2;
        return oz > 0 ? 5 : 4;
    }
    if (n == 2) {
        if (!oz) return edge_class(0, 1, ox, oy);
        if (!oy) return edge_class(0, 2, ox, oz);
        return edge_class(1, 2, oy, oz);
    }
    return -1;
}

// RouteTab index of the pure face pattern for face 0..5.
__host__ __device__ constexpr int face_pattern(int face) {
    return face == 0 ? 12 : face == 1 ? 14 : face == 2 ? 10 : face == 3 ? 16 : face == 4 ? 4 : 22;
}

// Error key: earliest iteration, then phase (every tile's P1 runs before any
// tile's P5 in the reference, engine.cpp:537-563), then lowest tile in
// coordinate order (the 1-worker reference order), then code.  atomicMin
// keeps the first.  Layout: iter << 37 | phase << 36 | tile_lin << 4 | code.
__device__ __forceinline__ void atomic_err(unsigned long long* err, long iter, int tile_lin,
                                           int code) {
    const unsigned long long phase = code == ERR_P5_NAN ? 1ull : 0ull;
    atomicMin(err, ((unsigned long long)iter << 37) | (phase << 36) |
                       ((unsigned long long)(unsigned)tile_lin << 4) | (unsigned)code);
}

// Extended-grid solid bit of the tile (local coords in [-1, E]).
template <int E>
__device__ __forceinline__ bool solid_at(const uint32_t* sb, int x, int y, int z) {
    constexpr int G = E + 2;
    const int idx = (x + 1) + G * ((y + 1) + G * (z + 1));
    return (sb[idx >> 5] >> (idx & 31)) & 1u;
}

// proj/src/scenario.cpp:177-183 — seed containment at cell centres.
__device__ __forceinline__ bool seed_contains(const SeedConst& s, double x, double y, double z) {
    if (s.shape == 0)
        return x >= s.lo[0] && x < s.hi[0] && y >= s.lo[1] && y < s.hi[1] && z >= s.lo[2] &&
               z < s.hi[2];
    const double dx = x - s.center[0], dy = y - s.center[1], dz = z - s.center[2];
    return dx * dx + dy * dy + dz * dz <= s.r2;
}

// The last seed of component c containing the cell centre (apply_seeds order,
// proj/src/engine.cpp:43-76), or -1.
template <int E>
__device__ __forceinline__ int seed_for(int c, const int* tc, int x, int y, int z) {
    int hit = -1;
    const double cx = double(tc[0] * E + x) + 0.5;
    const double cy = double(tc[1] * E + y) + 0.5;
    const double cz = double(tc[2] * E + z) + 0.5;
    for (int s = 0; s < P.n_seeds; ++s)
        if (P.seeds[s].comp == c && seed_contains(P.seeds[s], cx, cy, cz)) hit = s;
    return hit;
}

// Generated f_in for GEN tiles: seeded equilibrium or ambient (create_tile,
// proj/src/tilemap.cpp:132-140, then apply_seeds).  Also the velocity the
// reference holds for that cell before its first collision.
template <int E>
__device__ __forceinline__ void gen_fin(int mode, int c, const int* tc, int x, int y, int z,
                                        double* f, double& u0, double& u1, double& u2) {
    const int s = (mode == MODE_GEN_SEEDED) ? seed_for<E>(c, tc, x, y, z) : -1;
    if (s >= 0) {
#pragma unroll
        for (int i = 0; i < Q; ++i) f[i] = P.seeds[s].feq[i];
        u0 = P.seeds[s].u[0];
        u1 = P.seeds[s].u[1];
        u2 = P.seeds[s].u[2];
    } else {
#pragma unroll
        for (int i = 0; i < Q; ++i) f[i] = P.comp[c].feq_amb[i];
        u0 = u1 = u2 = 0.0;
    }
}

// Per-CTA routing table for each out pattern (ox+1)+3(oy+1)+9(oz+1): the
// source slot and the base pointer of that slot's block (buffer or psi faces).
// `nb` flags tiles born at the end of the previous step (GEN_AMBIENT): their
// psi faces are those of a fresh ambient cell, taken from the constants, so a
// peer rank never has to wait for a newborn's face buffer to be written.
struct RouteTab {
    int s[27];
    const double* p[27];
    uint8_t nb[27];
};
__device__ __forceinline__ void load_routes(RouteTab& rt, const int* routes, int self, int amb,
                                            double* const* bases, const uint8_t* mode = nullptr) {
    for (int k = threadIdx.x; k < 27; k += blockDim.x) {
        const int ox = k % 3 - 1, oy = (k / 3) % 3 - 1, oz = k / 9 - 1;
        const int cls = ghost_class(ox, oy, oz);
        const int s = (ox == 0 && oy == 0 && oz == 0) ? self : (cls < 0 ? amb : routes[cls]);
        rt.s[k] = s;
        rt.p[k] = bases[s];
        rt.nb[k] = mode ? uint8_t(mode[s] == MODE_GEN_AMBIENT) : uint8_t(0);
    }
}

// Pull of one cell's 19 populations of component c from f_post (the
// reference's P4a ghost fill + stream_pull, proj/src/kernels.cpp:5-30):
//   f_in[i](x) = solid(x - e_i) ? f_post(x)[opp i] : f_post(route(x - e_i))[i]
// `op(i, ptr)` receives each population's source address.  AA selects where
// the A-A storage kinds keep those values (see AA_LOCAL / AA_NEIGH above).
template <int E, int AA = AA_OFF, class Op>
__device__ __forceinline__ void pull_addr(const RouteTab& rt, int c, bool hs, const uint32_t* sb,
                                          int x, int y, int z, Op&& op) {
    constexpr int E3 = E * E * E;
    const size_t cs = size_t(Q) * E3;
    const int own = (z * E + y) * E + x;
#pragma unroll
    for (int i = 0; i < Q; ++i) {
        const int sx = x - ex_(i), sy = y - ey_(i), sz = z - ez_(i);
        const int ox = sx < 0 ? -1 : (sx >= E ? 1 : 0);
        const int oy = sy < 0 ? -1 : (sy >= E ? 1 : 0);
        const int oz = sz < 0 ? -1 : (sz >= E ? 1 : 0);
        const int pat = (ox + 1) + 3 * (oy + 1) + 9 * (oz + 1);
        const double* base = rt.p[pat];
        int cell = ((sz & (E - 1)) * E + (sy & (E - 1))) * E + (sx & (E - 1));
        int dir = i;
        if (hs && solid_at<E>(sb, sx, sy, sz)) {
            base = rt.p[13];
            cell = own;
            dir = AA == AA_OFF ? opp_(i) : i;
        } else if constexpr (AA != AA_OFF) {
            if (rt.s[pat] == P.amb_slot) {
                cell = own;  // feq_amb[i], any cell of the ambient slot
            } else if (AA == AA_LOCAL) {
                base = rt.p[13];
                cell = own;
            } else {
                dir = opp_(i);
            }
        }
        op(i, base + c * cs + size_t(dir) * E3 + cell);
    }
}

// A-A store address of f_post(x)[i] on an AA_NEIGH step: (x + e_i, i) in the
// geometric neighbour (rw = ROUTE_W table over the same buffer), (x, opp i)
// when x + e_i is solid, nullptr when the neighbour tile is absent.
template <int E>
__device__ __forceinline__ double* aa_push_addr(const RouteTab& rw, int c, bool hs, const uint32_t* sb,
                                                int x, int y, int z, int i) {
    constexpr int E3 = E * E * E;
    const size_t cs = size_t(Q) * E3;
    const int tx = x + ex_(i), ty = y + ey_(i), tz = z + ez_(i);
    if (hs && solid_at<E>(sb, tx, ty, tz))
        return const_cast<double*>(rw.p[13]) + c * cs + size_t(opp_(i)) * E3 + (z * E + y) * E + x;
    const int ox = tx < 0 ? -1 : (tx >= E ? 1 : 0);
    const int oy = ty < 0 ? -1 : (ty >= E ? 1 : 0);
    const int oz = tz < 0 ? -1 : (tz >= E ? 1 : 0);
    const int pat = (ox + 1) + 3 * (oy + 1) + 9 * (oz + 1);
    if (rw.s[pat] == P.amb_slot) return nullptr;
    return const_cast<double*>(rw.p[pat]) + c * cs + size_t(i) * E3 +
           ((tz & (E - 1)) * E + (ty & (E - 1))) * E + (tx & (E - 1));
}

// Store functor of one cell's 19 post-collision populations for a storage
// kind: A-B -> (x, i) of the output buffer; AA_LOCAL -> (x, opp i);
// AA_NEIGH -> aa_push_addr.  `own` = the cell's address for direction 0 in
// this component's block.
template <int E, int AA>
struct StoreF {
    double* own;
    const RouteTab* rw;
    int c, x, y, z;
    bool hs;
    const uint32_t* sb;
    // AA_NEIGH rows of a solid-free tile with z interior (warp-uniform): the
    // targets (x + e_i, i) from six precomputed bases (this row / the row
    // across the y edge, each with its x neighbours; nullptr = absent tile,
    // dropped); every row of such a plane takes it, so no warp lags behind
    // at the plane barrier.
    bool fast = false;
    double *xm = nullptr, *xp = nullptr, *yo = nullptr, *yxm = nullptr, *yxp = nullptr;
    __device__ __forceinline__ void operator()(int i, double v) const {
        constexpr int E2 = E * E;
        constexpr int E3 = E * E * E;
        if constexpr (AA == AA_OFF) {
            own[size_t(i) * E3] = v;
        } else if constexpr (AA == AA_LOCAL) {
            own[size_t(opp_(i)) * E3] = v;
        } else {
            if (fast) {
                const bool cy = (ey_(i) > 0 && y == E - 1) || (ey_(i) < 0 && y == 0);
                double* b;
                if (ex_(i) > 0) b = cy ? yxp : (x == E - 1 ? xp : own + 1);
                else if (ex_(i) < 0) b = cy ? yxm : (x == 0 ? xm : own - 1);
                else b = cy ? yo : own;
                if (b) b[i * E3 + ey_(i) * E + ez_(i) * E2] = v;
                return;
            }
            double* p = aa_push_addr<E>(*rw, c, hs, sb, x, y, z, i);
            if (p) *p = v;
        }
    }
};

// A-A pulls of a row of a solid-free tile with z interior (warp-uniform; any
// y): LOCAL reads (x, i), NEIGH reads (x - e_i, opp i); a source in an absent
// tile reads feq_amb[i] from the ambient slot.  Six bases as in
// pull_addr_fast_yedge (this row and the row across the y edge, with their
// x neighbours).
template <int E, int AA, class Op>
__device__ __forceinline__ void pull_addr_row_aa(const RouteTab& rt, int c, int x, int y, int z, Op&& op) {
    constexpr int E2 = E * E;
    constexpr int E3 = E * E * E;
    const size_t cs = size_t(Q) * E3;
    const int amb = P.amb_slot;
    const int row = (z * E + y) * E;
    const double* own = rt.p[13] + c * cs + row + x;
    const double* bp = x == 0 ? rt.p[12] + c * cs + row + (E - 1) : own - 1;
    const double* bm = x == E - 1 ? rt.p[14] + c * cs + row : own + 1;
    const bool ap = x == 0 && rt.s[12] == amb;
    const bool am = x == E - 1 && rt.s[14] == amb;
    const int oy = y == 0 ? -1 : 1;      // the row across the y edge (edge rows only)
    const int wrap = y == 0 ? E2 : -E2;
    const double* ownY = rt.p[13 + 3 * oy] + c * cs + row + x + wrap;
    const double* bpY = x == 0 ? rt.p[12 + 3 * oy] + c * cs + row + (E - 1) + wrap : ownY - 1;
    const double* bmY = x == E - 1 ? rt.p[14 + 3 * oy] + c * cs + row + wrap : ownY + 1;
    const bool aY = rt.s[13 + 3 * oy] == amb;
    const bool apY = x == 0 ? rt.s[12 + 3 * oy] == amb : aY;
    const bool amY = x == E - 1 ? rt.s[14 + 3 * oy] == amb : aY;
#pragma unroll
    for (int i = 0; i < Q; ++i) {
        const bool cy = (ey_(i) > 0 && y == 0) || (ey_(i) < 0 && y == E - 1);
        const double* b;
        bool a;
        if (ex_(i) > 0) { b = cy ? bpY : bp; a = cy ? apY : ap; }
        else if (ex_(i) < 0) { b = cy ? bmY : bm; a = cy ? amY : am; }
        else { b = cy ? ownY : own; a = cy && aY; }
        if constexpr (AA == AA_LOCAL) op(i, (a ? b : own) + size_t(i) * E3);
        else op(i, a ? b + size_t(i) * E3 : b + (opp_(i) * E3 - ey_(i) * E - ez_(i) * E2));
    }
}

// Fast pull for a cell whose y and z neighbours all lie inside the tile and
// whose tile has no solid cell (warp-uniform in callers: one warp = one x row).
// Only the x shift can leave the tile; that lane-dependent choice collapses to
// two base pointers, and every population is a load at a compile-time
// immediate offset from one of three bases.
template <int E, class Op>
__device__ __forceinline__ void pull_addr_fast(const RouteTab& rt, int c, int x, int y, int z,
                                               Op&& op) {
    constexpr int E2 = E * E;
    constexpr int E3 = E * E * E;
    const size_t cs = size_t(Q) * E3;
    const int row = (z * E + y) * E;
    const double* own = rt.p[13] + c * cs + row + x;
    // ex = +1 pulls from x-1: the -x neighbour's column E-1 on lane x == 0
    const double* bp = x == 0 ? rt.p[12] + c * cs + row + (E - 1) : own - 1;
    // ex = -1 pulls from x+1: the +x neighbour's column 0 on lane x == E-1
    const double* bm = x == E - 1 ? rt.p[14] + c * cs + row : own + 1;
#pragma unroll
    for (int i = 0; i < Q; ++i) {
        const int off = i * E3 - ey_(i) * E - ez_(i) * E2;
        const double* b = ex_(i) > 0 ? bp : (ex_(i) < 0 ? bm : own);
        op(i, b + off);
    }
}

// The same for a y-edge row (y == 0 or y == E-1; warp-uniform) of a tile with
// no solid cell, z interior: directions whose y shift leaves the tile read the
// -y / +y neighbour (rt.p 10 / 16, and the xy-diagonal tiles 9, 11 / 15, 17 on
// the x-edge lanes) at row E-1 / 0 — the addresses pull_addr computes, from
// three more base pointers instead of a per-direction route lookup.
template <int E, class Op>
__device__ __forceinline__ void pull_addr_fast_yedge(const RouteTab& rt, int c, int x, int y, int z,
                                                     Op&& op) {
    constexpr int E2 = E * E;
    constexpr int E3 = E * E * E;
    const size_t cs = size_t(Q) * E3;
    const int row = (z * E + y) * E;
    const double* own = rt.p[13] + c * cs + row + x;
    const double* bp = x == 0 ? rt.p[12] + c * cs + row + (E - 1) : own - 1;
    const double* bm = x == E - 1 ? rt.p[14] + c * cs + row : own + 1;
    const int oy = y == 0 ? -1 : 1;      // the neighbour row the crossing directions read
    const int wrap = y == 0 ? E2 : -E2;  // row -1 -> E-1, row E -> 0
    const double* ownY = rt.p[13 + 3 * oy] + c * cs + row + x + wrap;
    const double* bpY = x == 0 ? rt.p[12 + 3 * oy] + c * cs + row + (E - 1) + wrap : ownY - 1;
    const double* bmY = x == E - 1 ? rt.p[14 + 3 * oy] + c * cs + row + wrap : ownY + 1;
#pragma unroll
    for (int i = 0; i < Q; ++i) {
        const int off = i * E3 - ey_(i) * E - ez_(i) * E2;
        const bool cy = (ey_(i) > 0 && y == 0) || (ey_(i) < 0 && y == E - 1);
        const double* b = ex_(i) > 0 ? (cy ? bpY : bp) : (ex_(i) < 0 ? (cy ? bmY : bm) : (cy ? ownY : own));
        op(i, b + off);
    }
}

template <int E, int AA = AA_OFF>
__device__ __forceinline__ void pull_cell(const RouteTab& rt, int c, bool hs, const uint32_t* sb,
                                          int x, int y, int z, double* f) {
    pull_addr<E, AA>(rt, c, hs, sb, x, y, z, [&](int i, const double* p) { f[i] = __ldg(p); });
}
// The same with the storage kind chosen at run time (read-back, checks).
template <int E>
__device__ __forceinline__ void pull_cell_k(int kind, const RouteTab& rt, int c, bool hs,
                                            const uint32_t* sb, int x, int y, int z, double* f) {
    if (kind == AA_LOCAL) pull_cell<E, AA_LOCAL>(rt, c, hs, sb, x, y, z, f);
    else if (kind == AA_NEIGH) pull_cell<E, AA_NEIGH>(rt, c, hs, sb, x, y, z, f);
    else pull_cell<E>(rt, c, hs, sb, x, y, z, f);
}
template <int E>
__device__ __forceinline__ void pull_cell_fast(const RouteTab& rt, int c, int x, int y, int z,
                                               double* f) {
    pull_addr_fast<E>(rt, c, x, y, z, [&](int i, const double* p) { f[i] = __ldg(p); });
}

// f_in for any mode (u is only meaningful for GEN modes).
template <int E, int AA = AA_OFF>
__device__ __forceinline__ void fin_cell(const RouteTab& rt, int mode, const int* tc, int c,
                                         bool hs, const uint32_t* sb, int x, int y, int z,
                                         double* f, double& u0, double& u1, double& u2) {
    if (mode == MODE_PULL) pull_cell<E, AA>(rt, c, hs, sb, x, y, z, f);
    else gen_fin<E>(mode, c, tc, x, y, z, f, u0, u1, u2);
}

// Face-layer index helpers: face f = 2*axis + (dir > 0); the in-face index
// uses the two remaining coordinates in increasing axis order.
template <int E>
__device__ __forceinline__ int face_index(int face, int x, int y, int z) {
    const int axis = face >> 1;
    return axis == 0 ? (y + E * z) : (axis == 1 ? (x + E * z) : (x + E * y));
}

// psi at an out-of-tile cell (local coords with 1 or 2 axes outside) from the
// routed tile's face buffer (P2 ghost fill, proj/src/engine.cpp:317-352).
// rt.p holds the psi-face bases of the ROUTE_PSI table.
template <int E>
__device__ __forceinline__ double psi_ghost(const RouteTab& rt, int c, bool hs, const uint32_t* sb,
                                            int x, int y, int z) {
    if (hs && solid_at<E>(sb, x, y, z)) return 0.0;
    const int ox = x < 0 ? -1 : (x >= E ? 1 : 0);
    const int oy = y < 0 ? -1 : (y >= E ? 1 : 0);
    const int oz = z < 0 ? -1 : (z >= E ? 1 : 0);
    const int pat = (ox + 1) + 3 * (oy + 1) + 9 * (oz + 1);
    if (rt.nb[pat]) return P.comp[c].psi_nb;
    const double* base = rt.p[pat];
    // the cell lies on the routed tile's face opposite our first out axis
    int face;
    if (ox) face = ox > 0 ? 0 : 1;
    else if (oy) face = oy > 0 ? 2 : 3;
    else face = oz > 0 ? 4 : 5;
    const int lx = x & (E - 1), ly = y & (E - 1), lz = z & (E - 1);
    constexpr int E2 = E * E;
    return base[(size_t(c) * 6 + face) * E2 + face_index<E>(face, lx, ly, lz)];
}

// ---------------------------------------------------------------------------
// k_main: the plain fused kernel (variant 1).  One CTA = one tile x one z-chunk
// of BZ planes x one y-chunk of YB rows; psi planes (with halo planes and rows
// recomputed) in a shared ring, and every population pulled twice (psi pass +
// collide).  Used for E = 8, E = 64 (YB = 16: the whole-plane ring would not
// fit shared memory) and psi-free scenarios (NOPSI: no pseudo-potential
// stencil at all — a single pull-collide pass per cell).  A-A storage (AA !=
// AA_OFF) needs the whole tile in one CTA (BZ = YB = E): recomputed halo
// planes / rows would read cells another CTA updates in place.
template <int E, int C, int BZ, int NT, bool NOPSI, int YB = E, int AA = AA_OFF>
__global__ void __launch_bounds__(NT) k_main(Dev d, const int* __restrict__ active, int src_buf,
                                             int write_uface, long iter) {
    static_assert(AA == AA_OFF || (BZ == E && YB == E), "A-A needs one CTA per tile");
    if (halted(d)) return;
    constexpr int G = E + 2;
    constexpr int GG = G * (YB + 2);  // one psi plane of the chunk incl. its halo
    constexpr int E2 = E * E;
    constexpr int E3 = E * E * E;
    constexpr int NZC = E / BZ;
    constexpr int NYC = E / YB;
    constexpr int CPT = (E * YB + NT - 1) / NT;          // cells per thread per plane
    constexpr int PPT = (E * (YB + 2) + NT - 1) / NT;    // psi positions per thread (x inside)
    extern __shared__ double smem[];
    double* psi = smem;  // [3][C][GG] ring of planes (unused when NOPSI)
    __shared__ RouteTab rt_pull, rt_psi, rt_w;
    __shared__ uint32_t s_solid[(G * G * G + 31) / 32];
    __shared__ int s_tc[3];

    if (d.nactive && d.tile_base + int(blockIdx.x / (NZC * NYC)) >= *d.nactive) return;
    const int slot = active[blockIdx.x / (NZC * NYC)];
    if (d.no_fluid && d.no_fluid[slot]) return;  // (see Dev::no_fluid)
    const int z0 = (blockIdx.x % NZC) * BZ;
    const int y0 = ((blockIdx.x / NZC) % NYC) * YB;
    const uint8_t mode = d.mode[slot];
    const bool hs = d.has_solid[slot] != 0;
    const int amb = P.amb_slot;
    const int par = int(iter & 1);
    double* __restrict__ fo = d.slot_f[src_buf ^ 1][slot];
    const int li = d.lidx[slot];
    load_routes(rt_pull, d.route[ROUTE_PULL] + size_t(slot) * 18, slot, amb, d.slot_f[src_buf]);
    load_routes(rt_psi, d.route[ROUTE_PSI] + size_t(slot) * 18, slot, amb, d.slot_pf[par], d.mode);
    if constexpr (AA == AA_NEIGH) load_routes(rt_w, d.route[ROUTE_W] + size_t(slot) * 18, slot, amb, d.slot_f[0]);
    if (threadIdx.x < 3) s_tc[threadIdx.x] = d.coords[slot * 3 + threadIdx.x];
    if (hs)
        for (int k = threadIdx.x; k < d.solid_words; k += NT)
            s_solid[k] = d.solid[size_t(slot) * d.solid_words + k];
    __syncthreads();
    const int tile_lin = (s_tc[0] * P.grid[1] + s_tc[1]) * P.grid[2] + s_tc[2];

    // ---- psi of plane pz (ring slot r) on rows y0-1 .. y0+YB incl. the x
    // ghost columns (rows outside the tile are ghost rows) ---------------------
    auto psi_plane = [&](int pz) {
        const int r = (pz + 3) % 3;
        const bool inside = pz >= 0 && pz < E;
        const bool zowned = pz >= z0 && pz < z0 + BZ;
        int negs = 0, clamps = 0;  // per-thread tallies, reduced per warp below
#pragma unroll 1
        for (int k = 0; k < PPT; ++k) {
            const int idx = threadIdx.x + k * NT;
            if (idx >= E * (YB + 2)) break;
            const int x = idx % E, y = y0 - 1 + idx / E;
            const bool owned = zowned && y >= y0 && y < y0 + YB;
#pragma unroll
            for (int c = 0; c < C; ++c) {
                double v = 0.0;
                if (!inside || y < 0 || y >= E) {
                    v = psi_ghost<E>(rt_psi, c, hs, s_solid, x, y, pz);
                } else if (!(hs && solid_at<E>(s_solid, x, y, pz))) {
                    double f[Q], u0, u1, u2;
                    fin_cell<E, AA>(rt_pull, mode, s_tc, c, hs, s_solid, x, y, pz, f, u0, u1, u2);
                    apply_pokes<E>(d, slot, c, x, y, pz, f);
                    double rho = 0.0;
#pragma unroll
                    for (int i = 0; i < Q; ++i) {
                        rho += f[i];
                        if (owned && f[i] < 0.0) ++negs;
                    }
                    const CompConst& kc = P.comp[c];
                    if (!isfinite(rho)) {
                        atomic_err(d.err, iter, tile_lin, ERR_P1_NAN);
                    } else {
                        double press;
                        if (!pr_pressure(rho, kc, press)) {
                            atomic_err(d.err, iter, tile_lin, ERR_P1_POLE);
                        } else {
                            bool cl;
                            v = pseudo_potential(rho, press, kc, cl);
                            if (owned && cl) ++clamps;
                        }
                    }
                }
                psi[(r * C + c) * GG + (x + 1) + G * (y - y0 + 1)] = v;
            }
        }
        // x ghost columns of rows y0-1 .. y0+YB: 2 (YB+2) positions
        for (int k = threadIdx.x; k < 2 * (YB + 2); k += NT) {
            const int x = k < YB + 2 ? -1 : E;
            const int y = y0 - 1 + (k < YB + 2 ? k : k - (YB + 2));
            const bool corner3 = !inside && (y < 0 || y >= E);
#pragma unroll
            for (int c = 0; c < C; ++c)
                psi[(r * C + c) * GG + (x + 1) + G * (y - y0 + 1)] =
                    corner3 ? 0.0 : psi_ghost<E>(rt_psi, c, hs, s_solid, x, y, pz);
        }
        if (zowned) {
            const unsigned m1 = __reduce_add_sync(0xffffffffu, (unsigned)negs);
            const unsigned m2 = __reduce_add_sync(0xffffffffu, (unsigned)clamps);
            if ((threadIdx.x & 31) == 0) {
                if (m1) atomicAdd(&d.cnt[CNT_NEG], (unsigned long long)m1);
                if (m2) atomicAdd(&d.cnt[CNT_CLAMP], (unsigned long long)m2);
            }
        }
    };

    // ---- collide plane z ----------------------------------------------------
    auto collide_plane = [&](int z) {
        int zero_rho = 0;
        int negs = 0;
        int suspect = 0;
#pragma unroll 1
        for (int k = 0; k < CPT; ++k) {
            const int idx = threadIdx.x + k * NT;
            if (idx >= E * YB) break;
            const int x = idx % E, y = y0 + idx / E;
            if (hs && solid_at<E>(s_solid, x, y, z)) continue;
            const int cell = (z * E + y) * E + x;
            const int rc = (z + 3) % 3, rm = (z + 2) % 3, rp = (z + 4) % 3;
            const int pc = (x + 1) + G * (y - y0 + 1);
#pragma unroll 1
            for (int c = 0; c < C; ++c) {
                double f[Q];
                double u0 = 0.0, u1 = 0.0, u2 = 0.0, rho;
                fin_cell<E, AA>(rt_pull, mode, s_tc, c, hs, s_solid, x, y, z, f, u0, u1, u2);
                apply_pokes<E>(d, slot, c, x, y, z, f);
                if (mode == MODE_PULL) {
                    moments(f, rho, u0, u1, u2);
                } else {
                    rho = sum19(f);  // P1 density; u is the stored seed/ambient u
                }
                if constexpr (NOPSI) {
                    // P1 tallies folded in: psi is +-0 (no clamps, no pole), so
                    // only the negative-population count and the NaN check remain.
#pragma unroll
                    for (int i = 0; i < Q; ++i) negs += f[i] < 0.0;
                    if (!isfinite(rho)) atomic_err(d.err, iter, tile_lin, ERR_P1_NAN);
                }
                const CompConst& kc = P.comp[c];
                // ---- force: gravity + intra + inter (engine.cpp:426-448)
                double F0 = 0.0, F1 = 0.0, F2 = 0.0;
                if (kc.has_gravity) {
                    F0 = rho * kc.gravity[0];
                    F1 = rho * kc.gravity[1];
                    F2 = rho * kc.gravity[2];
                }
                if constexpr (!NOPSI) {
                    // intra_force, proj/src/physics.cpp:44-63
                    const double* pm = psi + (rm * C + c) * GG + pc;
                    const double* p0 = psi + (rc * C + c) * GG + pc;
                    const double* pp = psi + (rp * C + c) * GG + pc;
                    double s10 = 0.0, s11 = 0.0, s12 = 0.0, s20 = 0.0, s21 = 0.0, s22 = 0.0;
#pragma unroll
                    for (int i = 1; i < Q; ++i) {
                        const int dx = ex_(i), dy = ey_(i), dz = ez_(i);
                        const double* pl = dz < 0 ? pm : (dz > 0 ? pp : p0);
                        const double pn = pl[dx + G * dy];
                        const double a1 = w_(i) * pn;
                        const double a2 = a1 * pn;
                        if (dx > 0) { s10 += a1; s20 += a2; }
                        if (dx < 0) { s10 -= a1; s20 -= a2; }
                        if (dy > 0) { s11 += a1; s21 += a2; }
                        if (dy < 0) { s11 -= a1; s21 -= a2; }
                        if (dz > 0) { s12 += a1; s22 += a2; }
                        if (dz < 0) { s12 -= a1; s22 -= a2; }
                    }
                    const double c1 = kc.c1f * p0[0];
                    const double c2 = kc.c2;
                    F0 += c1 * s10 + c2 * s20;
                    F1 += c1 * s11 + c2 * s21;
                    F2 += c1 * s12 + c2 * s22;
                    // inter_force, proj/src/physics.cpp:65-78
#pragma unroll
                    for (int c2i = 0; c2i < C; ++c2i) {
                        if (c2i == c) continue;
                        const double g = P.coupling[c * C + c2i];
                        if (g == 0.0) continue;
                        const double* qm = psi + (rm * C + c2i) * GG + pc;
                        const double* q0 = psi + (rc * C + c2i) * GG + pc;
                        const double* qp = psi + (rp * C + c2i) * GG + pc;
                        double t0 = 0.0, t1 = 0.0, t2 = 0.0;
#pragma unroll
                        for (int i = 1; i < Q; ++i) {
                            const int dx = ex_(i), dy = ey_(i), dz = ez_(i);
                            const double* pl = dz < 0 ? qm : (dz > 0 ? qp : q0);
                            const double a1 = w_(i) * pl[dx + G * dy];
                            if (dx > 0) t0 += a1;
                            if (dx < 0) t0 -= a1;
                            if (dy > 0) t1 += a1;
                            if (dy < 0) t1 -= a1;
                            if (dz > 0) t2 += a1;
                            if (dz < 0) t2 -= a1;
                        }
                        const double cc = (-g) * p0[0];
                        F0 += cc * t0;
                        F1 += cc * t1;
                        F2 += cc * t2;
                    }
                } else {
                    // psi == +-0: the intra/inter terms are signed zeros
                    F0 += 0.0;
                    F1 += 0.0;
                    F2 += 0.0;
                }
                // ---- u_prev bookkeeping for the criterion / capture
                if (write_uface) {
#pragma unroll
                    for (int face = 0; face < 6; ++face) {
                        const int axis = face >> 1;
                        const int coord = axis == 0 ? x : (axis == 1 ? y : z);
                        if (coord == ((face & 1) ? E - 1 : 0) && rt_psi.s[face_pattern(face)] == amb) {
                            double* uf = d.u_face + ((size_t(li) * C + c) * 6 + face) * 3 * E2;
                            const int fi = face_index<E>(face, x, y, z);
                            uf[fi] = u0;
                            uf[E2 + fi] = u1;
                            uf[2 * E2 + fi] = u2;
                        }
                    }
                }
                if (d.capture) {
                    double* cp = d.capture + (size_t(li) * C + c) * 4 * E3;
                    // psi-free: radicand 2(+0)/(cs2 g) is a signed zero, sqrt keeps it
                    cp[cell] = NOPSI ? (kc.cs2_g < 0.0 ? -0.0 : 0.0) : psi[(rc * C + c) * GG + pc];
                    cp[E3 + cell] = u0;
                    cp[2 * E3 + cell] = u1;
                    cp[3 * E3 + cell] = u2;
                }
                // ---- collision (engine.cpp:450-475)
                const double om = kc.omega;
                const StoreF<E, AA> out{fo + c * size_t(Q) * E3 + cell, &rt_w, c, x, y, z, hs, s_solid};
                const double uu = u0 * u0 + u1 * u1 + u2 * u2;
                const double t3 = (0.5 * uu) * 3.0;
                const double wr0 = PLBM_W0 * rho, wr1 = PLBM_W1 * rho, wr2 = PLBM_W2 * rho;
                const bool unforced = (F0 == 0.0 && F1 == 0.0 && F2 == 0.0);
                if (!unforced && rho <= 0.0) ++zero_rho;
                Screen scr;
                if (unforced || rho <= 0.0) {
#define PLBM_RELAX(I)                                                                 \
    {                                                                                 \
        const double wr = (I == 0) ? wr0 : ((I <= 6) ? wr1 : wr2);                    \
        const double eu = (I == 0) ? 0.0 : eu_pair<(I == 0 ? 1 : I - ((I + 1) & 1))>(u0, u1, u2); \
        const double e0 = feq_dir<I>(wr, eu, t3);                                     \
        const double o_ = f[I] + om * (e0 - f[I]);                                     \
        out(I, o_);                                                                   \
        scr.add(o_);                                                                  \
    }
                    PLBM_RELAX(0) PLBM_RELAX(1) PLBM_RELAX(2) PLBM_RELAX(3) PLBM_RELAX(4)
                    PLBM_RELAX(5) PLBM_RELAX(6) PLBM_RELAX(7) PLBM_RELAX(8) PLBM_RELAX(9)
                    PLBM_RELAX(10) PLBM_RELAX(11) PLBM_RELAX(12) PLBM_RELAX(13) PLBM_RELAX(14)
                    PLBM_RELAX(15) PLBM_RELAX(16) PLBM_RELAX(17) PLBM_RELAX(18)
#undef PLBM_RELAX
                } else {
                    const double v0 = u0 + F0 / rho, v1 = u1 + F1 / rho, v2 = u2 + F2 / rho;
                    const double vv = v0 * v0 + v1 * v1 + v2 * v2;
                    const double s3 = (0.5 * vv) * 3.0;
#define PLBM_FORCED(I)                                                                \
    {                                                                                 \
        constexpr int IP = (I == 0 ? 1 : I - ((I + 1) & 1));                          \
        const double wr = (I == 0) ? wr0 : ((I <= 6) ? wr1 : wr2);                    \
        const double eu = (I == 0) ? 0.0 : eu_pair<IP>(u0, u1, u2);                   \
        const double ev = (I == 0) ? 0.0 : eu_pair<IP>(v0, v1, v2);                   \
        const double e0 = feq_dir<I>(wr, eu, t3);                                     \
        const double e1 = feq_dir<I>(wr, ev, s3);                                     \
        const double o_ = f[I] + ((om * (e0 - f[I]) + e1) - e0);                       \
        out(I, o_);                                                                   \
        scr.add(o_);                                                                  \
    }
                    PLBM_FORCED(0) PLBM_FORCED(1) PLBM_FORCED(2) PLBM_FORCED(3) PLBM_FORCED(4)
                    PLBM_FORCED(5) PLBM_FORCED(6) PLBM_FORCED(7) PLBM_FORCED(8) PLBM_FORCED(9)
                    PLBM_FORCED(10) PLBM_FORCED(11) PLBM_FORCED(12) PLBM_FORCED(13)
                    PLBM_FORCED(14) PLBM_FORCED(15) PLBM_FORCED(16) PLBM_FORCED(17)
                    PLBM_FORCED(18)
#undef PLBM_FORCED
                }
                suspect |= scr.suspect();
            }
        }
        const unsigned zr = __reduce_add_sync(0xffffffffu, (unsigned)zero_rho);
        if ((threadIdx.x & 31) == 0 && zr) atomicAdd(&d.cnt[CNT_ZERO_RHO], (unsigned long long)zr);
        if (__any_sync(0xffffffffu, suspect) && (threadIdx.x & 31) == 0) {
            d.suspect[slot] = 1;
            if (d.susp_any) atomicOr(&d.susp_any[iter & 1], 1u);
        }
        if constexpr (NOPSI) {
            const unsigned ng = __reduce_add_sync(0xffffffffu, (unsigned)negs);
            if ((threadIdx.x & 31) == 0 && ng) atomicAdd(&d.cnt[CNT_NEG], (unsigned long long)ng);
        }
    };

    if constexpr (NOPSI) {
        (void)psi;
#pragma unroll 1
        for (int z = z0; z < z0 + BZ; ++z) collide_plane(z);
    } else {
        psi_plane(z0 - 1);
        psi_plane(z0);
#pragma unroll 1
        for (int z = z0; z < z0 + BZ; ++z) {
            psi_plane(z + 1);
            __syncthreads();
            collide_plane(z);
            __syncthreads();
        }
    }
}

// ---------------------------------------------------------------------------
// Face pass (P5 moments of f_in^(k+1) on the six face layers): per face cell
// and component, pull f_in^(k+1), psi for the next step's ghost faces, the P5
// NaN check (engine.cpp:509-512) and, on a frontier face, the activation
// criterion (tilemap.cpp:182-218).  Work items are (face cell, component)
// pairs; with PF each thread prefetches its next item's 19 populations before
// it finishes the current one (two items in flight per thread, 126 registers);
// without PF one item is in flight and occupancy supplies the parallelism (the
// standalone k_face runs that way at 4 CTAs/SM, measured 0.216 vs 0.245 ms).
// Faces 6.. ("mid faces", Dev::mid_faces): face 6 + 2 (b - 1) + s is the row
// y = b * P.mid_sp - 1 + s inside the tile (s = 0 below the boundary, 1
// above), in-face index x + E z like the y faces.
__device__ __forceinline__ int mid_face_row(int face) { return ((face - 6) / 2 + 1) * P.mid_sp - 1 + (face & 1); }
template <int E>
__device__ __forceinline__ void face_xyz(int face, int idx, int& x, int& y, int& z) {
    if (face >= 6) {
        x = idx % E;
        y = mid_face_row(face);
        z = idx / E;
        return;
    }
    const int axis = face >> 1;
    const int fixed = (face & 1) ? E - 1 : 0;
    const int a = idx % E, b = idx / E;
    x = axis == 0 ? fixed : a;
    y = axis == 0 ? a : (axis == 1 ? fixed : b);
    z = axis == 2 ? fixed : b;
}

// COH: read f_post through L2 (written by other CTAs of the same launch in
// the fused path).
template <int E, bool COH>
__device__ __forceinline__ void face_load(const RouteTab& rt, int mode, const int* tc, int c, bool hs,
                                          const uint32_t* sb, int face, int idx, double* f,
                                          bool xcol = false, int kind = AA_OFF) {
    int x, y, z;
    face_xyz<E>(face, idx, x, y, z);
    if (hs && solid_at<E>(sb, x, y, z)) return;
    // x faces from the xcol side buffers (below) whatever the storage kind:
    // they hold f_post of the boundary columns, i.e. the values the A-B pull
    // rule reads, which is f_in of the next step under A-A storage too
    if (kind != AA_OFF && !(xcol && face < 2 && !hs && mode == MODE_PULL)) {  // A-A: general addressing
        if (mode != MODE_PULL) {
            double a0, a1, a2;
            gen_fin<E>(mode, c, tc, x, y, z, f, a0, a1, a2);
        } else if (kind == AA_LOCAL) {
            pull_addr<E, AA_LOCAL>(rt, c, hs, sb, x, y, z, [&](int i, const double* p) { f[i] = COH ? __ldcg(p) : __ldg(p); });
        } else {
            pull_addr<E, AA_NEIGH>(rt, c, hs, sb, x, y, z, [&](int i, const double* p) { f[i] = COH ? __ldcg(p) : __ldg(p); });
        }
        return;
    }
    if (xcol && face < 2 && !hs && mode == MODE_PULL) {
        // x faces from the routed tiles' xcol buffers (lattice.cuh): the
        // source column x - e_x is 0 / 1 / E-2 / E-1 of the own tile or x = E-1
        // / 0 of the -x / +x neighbour; consecutive threads read consecutive y
        constexpr int E2 = E * E;
        constexpr int E3 = E * E * E;
#pragma unroll
        for (int i = 0; i < Q; ++i) {
            const int sx = x - ex_(i), sy = y - ey_(i), sz = z - ez_(i);
            const int ox = sx < 0 ? -1 : (sx >= E ? 1 : 0);
            const int oy = sy < 0 ? -1 : (sy >= E ? 1 : 0);
            const int oz = sz < 0 ? -1 : (sz >= E ? 1 : 0);
            const int lx = sx & (E - 1);
            const int cls = lx == 0 ? 0 : lx == 1 ? 1 : lx == E - 2 ? 2 : 3;
            const double* p = rt.p[(ox + 1) + 3 * (oy + 1) + 9 * (oz + 1)] + size_t(P.C) * Q * E3 +
                              (size_t(c) * XN + xslot_sel(cls, i)) * E2 + (sz & (E - 1)) * E + (sy & (E - 1));
            f[i] = COH ? __ldcg(p) : __ldg(p);
        }
        return;
    }
    if (mode == MODE_PULL && !hs && face >= 6 && z >= 1 && z <= E - 2) {  // mid faces: interior rows
        if (COH) pull_addr_fast<E>(rt, c, x, y, z, [&](int i, const double* p) { f[i] = __ldcg(p); });
        else pull_addr_fast<E>(rt, c, x, y, z, [&](int i, const double* p) { f[i] = __ldg(p); });
        return;
    }
    if (mode == MODE_PULL && !hs && (face == 2 || face == 3) && z >= 1 && z <= E - 2) {
        // y faces: the tile-edge-row fast pull (no per-direction route lookup)
        if (COH) pull_addr_fast_yedge<E>(rt, c, x, y, z, [&](int i, const double* p) { f[i] = __ldcg(p); });
        else pull_addr_fast_yedge<E>(rt, c, x, y, z, [&](int i, const double* p) { f[i] = __ldg(p); });
        return;
    }
    if (mode == MODE_PULL) {
        if (COH) pull_addr<E>(rt, c, hs, sb, x, y, z, [&](int i, const double* p) { f[i] = __ldcg(p); });
        else pull_addr<E>(rt, c, hs, sb, x, y, z, [&](int i, const double* p) { f[i] = __ldg(p); });
    } else {
        double a0, a1, a2;
        gen_fin<E>(mode, c, tc, x, y, z, f, a0, a1, a2);
    }
}

// Returns true when the criterion fires at this cell.
template <int E>
__device__ __forceinline__ bool face_finish(const Dev& d, int mode, int c, bool hs, const uint32_t* sb,
                                            int face, int idx, const double* f, bool frontier,
                                            bool nan_check, int li, double* pf, long iter, int tile_lin) {
    constexpr int E2 = E * E;
    int x, y, z;
    face_xyz<E>(face, idx, x, y, z);
    bool fired = false;
    double v = 0.0;
    if (!(hs && solid_at<E>(sb, x, y, z))) {
        double rho = 0.0;
#pragma unroll
        for (int i = 0; i < Q; ++i) rho += f[i];
        if (mode == MODE_PULL && (frontier || nan_check)) {
            // u = m / rho (kernels.hpp:31-48) is needed for the criterion; for
            // the NaN check alone it is provably finite when |m| <= 2^100 and
            // |rho| >= 2^-900, so the divisions are skipped then
            double m0 = 0.0, m1 = 0.0, m2 = 0.0;
            m0 += f[1]; m0 -= f[2]; m0 += f[7]; m0 -= f[8]; m0 += f[9]; m0 -= f[10];
            m0 += f[11]; m0 -= f[12]; m0 += f[13]; m0 -= f[14];
            m1 += f[3]; m1 -= f[4]; m1 += f[7]; m1 -= f[8]; m1 -= f[9]; m1 += f[10];
            m1 += f[15]; m1 -= f[16]; m1 += f[17]; m1 -= f[18];
            m2 += f[5]; m2 -= f[6]; m2 += f[11]; m2 -= f[12]; m2 -= f[13]; m2 += f[14];
            m2 += f[15]; m2 -= f[16]; m2 -= f[17]; m2 += f[18];
            const bool safe = fabs(rho) >= 0x1p-900 && fabs(m0) <= 0x1p100 && fabs(m1) <= 0x1p100 &&
                              fabs(m2) <= 0x1p100;
            double u0 = 0.0, u1 = 0.0, u2 = 0.0;
            if ((frontier || !safe) && rho != 0.0) {
                u0 = m0 / rho;
                u1 = m1 / rho;
                u2 = m2 / rho;
            }
            if (nan_check && (!isfinite(rho) ||
                              (!safe && (!isfinite(u0) || !isfinite(u1) || !isfinite(u2)))))
                atomic_err(d.err, iter, tile_lin, ERR_P5_NAN);
            if (frontier) {
                const double* uf = d.u_face + ((size_t(li) * P.C + c) * 6 + face) * 3 * E2;
                const double dx = u0 - __ldcg(uf + idx), dy = u1 - __ldcg(uf + E2 + idx),
                             dz = u2 - __ldcg(uf + 2 * E2 + idx);
                if (dx * dx + dy * dy + dz * dz > P.s2) fired = true;
            }
        } else if (nan_check && !isfinite(rho)) {
            atomic_err(d.err, iter, tile_lin, ERR_P5_NAN);
        }
        double press;
        if (isfinite(rho) && pr_pressure(rho, P.comp[c], press)) {
            bool cl;
            v = pseudo_potential(rho, press, P.comp[c], cl);
        }
    }
    pf[(face < 6 ? size_t(c) * 6 + face : size_t(P.C) * 6 + size_t(c) * d.mid_faces + (face - 6)) * E2 + idx] = v;
    return fired;
}

// Items t = 0, 1, ... of this thread: cell k = k0 + tid + (t / nc) * NT of
// the 6 E^2 face cells (k < k1), component c0 + t % nc.  Returns the bitmask
// of faces whose criterion fired (OR over the warp, set by lane 0 only).
template <int E, int NT, bool COH, bool PF = true>
__device__ unsigned face_run(const Dev& d, const RouteTab& rt, int mode, const int* tc, bool hs,
                             const uint32_t* sb, int c0, int nc, int k0, int k1, const int* routes,
                             bool criterion, bool nan_check, int li, double* pf, long iter,
                             int tile_lin) {
    constexpr int E2 = E * E;
    unsigned fired = 0;
    auto item = [&](int t, int& face, int& idx, int& c) {
        const int k = k0 + int(threadIdx.x) + (t / nc) * NT;
        if (k >= k1) return false;
        face = k / E2;
        idx = k - face * E2;
        c = c0 + t % nc;
        return true;
    };
    const bool xcol = d.xcol_ok != 0;
    const int kind = aa_kind(d.aa, iter + 1);  // the storage kind the next step reads
    auto load = [&](int t, double* f) {
        int face, idx, c;
        if (item(t, face, idx, c)) face_load<E, COH>(rt, mode, tc, c, hs, sb, face, idx, f, xcol, kind);
    };
    auto finish = [&](int t, const double* f) {
        int face, idx, c;
        if (!item(t, face, idx, c)) return false;
        const bool frontier = criterion && face < 6 && routes[face] == P.amb_slot && !(fired & (1u << face));
        if (face_finish<E>(d, mode, c, hs, sb, face, idx, f, frontier, nan_check && face < 6, li, pf, iter,
                           tile_lin))
            fired |= 1u << face;
        return true;
    };
    if constexpr (PF) {
        double fa[Q], fb[Q];
        load(0, fa);
#pragma unroll 1
        for (int t = 0;; t += 2) {
            load(t + 1, fb);
            if (!finish(t, fa)) break;
            load(t + 2, fa);
            if (!finish(t + 1, fb)) break;
        }
    } else {
        double fa[Q];
#pragma unroll 1
        for (int t = 0;; ++t) {
            load(t, fa);
            if (!finish(t, fa)) break;
        }
    }
    return __reduce_or_sync(0xffffffffu, fired);
}

__device__ __forceinline__ void set_triggers(const Dev& d, int slot, unsigned faces) {
    if (faces && (threadIdx.x & 31) == 0)
        atomicOr((unsigned*)(d.trig) + slot / 4, faces << (8 * (slot % 4)));
}

// The face pass of tile `slot`, components [c0, c0 + nc), face cells [k0, k1),
// run by one CTA inside the fused kernel once the tile's dependencies are
// complete.  rt / sb / tc are the CTA's shared scratch.
template <int E, int NT>
__device__ void face_pass_part(const Dev& d, int slot, int c0, int nc, int k0, int k1, int post_buf,
                               long iter, RouteTab& rt, uint32_t* sb, int* tc) {
    __syncthreads();  // the shared scratch is free
    load_routes(rt, d.route[ROUTE_PSI] + size_t(slot) * 18, slot, P.amb_slot, d.slot_f[post_buf]);
    const bool hs = d.has_solid[slot] != 0;
    if (hs)
        for (int k = threadIdx.x; k < d.solid_words; k += NT) sb[k] = d.solid[size_t(slot) * d.solid_words + k];
    if (threadIdx.x < 3) tc[threadIdx.x] = d.coords[slot * 3 + threadIdx.x];
    __syncthreads();
    const int tile_lin = (tc[0] * P.grid[1] + tc[1]) * P.grid[2] + tc[2];
    const unsigned f = face_run<E, NT, true>(
        d, rt, MODE_PULL, tc, hs, sb, c0, nc, k0, k1, d.route[ROUTE_PSI] + size_t(slot) * 18,
        (d.face_flags & FACE_CRITERION) != 0, (d.face_flags & FACE_NAN) != 0, d.lidx[slot],
        d.slot_pf[int((iter + 1) & 1)][slot], iter, tile_lin);
    set_triggers(d, slot, f);
}

// k_face: the face pass as its own launch (multi-rank runs, the non-fused
// kernels, and the initial psi faces).  One CTA per (tile, face).
template <int E, int C, int NT, int MINB = 1, bool PF = true>
__global__ void __launch_bounds__(NT, MINB) k_face(Dev d, const int* __restrict__ active, int src_buf,
                                             int flags, long iter) {
    if (halted(d)) return;
    constexpr int E2 = E * E;
    constexpr int G = E + 2;
    __shared__ RouteTab rt;
    __shared__ uint32_t s_solid[(G * G * G + 31) / 32];
    __shared__ int s_tc[3];
    const int nf = 6 + d.mid_faces;
    if (d.nactive && d.tile_base + int(blockIdx.x / nf) >= *d.nactive) return;
    const int slot = active[blockIdx.x / nf];
    if (d.no_fluid && d.no_fluid[slot]) return;  // (see Dev::no_fluid)
    const int face = blockIdx.x % nf;
    const uint8_t mode = d.mode[slot];
    const bool hs = d.has_solid[slot] != 0;
    // after k_main every tile pulls with the map it just stepped on (ROUTE_PSI)
    load_routes(rt, d.route[ROUTE_PSI] + size_t(slot) * 18, slot, P.amb_slot, d.slot_f[src_buf]);
    if (threadIdx.x < 3) s_tc[threadIdx.x] = d.coords[slot * 3 + threadIdx.x];
    if (hs)
        for (int k = threadIdx.x; k < d.solid_words; k += NT)
            s_solid[k] = d.solid[size_t(slot) * d.solid_words + k];
    __syncthreads();
    const int tile_lin = (s_tc[0] * P.grid[1] + s_tc[1]) * P.grid[2] + s_tc[2];
    const unsigned f = face_run<E, NT, false, PF>(d, rt, mode, s_tc, hs, s_solid, 0, C, face * E2,
                                              (face + 1) * E2, d.route[ROUTE_PSI] + size_t(slot) * 18,
                                              (flags & 1) != 0, (flags & 2) != 0, d.lidx[slot],
                                              d.slot_pf[int((iter + 1) & 1)][slot], iter, tile_lin);
    set_triggers(d, slot, f);
}

// k_p5: the exact P5 check (proj/src/engine.cpp:500-512: moments of every
// fluid cell of the post-stream state, EngineError(it, tile, "P5") on a
// non-finite rho or u) for the tiles the fused kernel's screen marked suspect
// (lattice.cuh Screen: an unmarked tile provably has finite moments).  Runs
// after the face pass of step `iter`, before that step's expansion; one CTA
// per tile, an unmarked tile exits at once.  Clears the marks it consumes.
template <int E, int C, int NT>
__global__ void __launch_bounds__(NT) k_p5(Dev d, const int* __restrict__ active, int src_buf, long iter) {
    if (halted(d)) return;
    // step iter-1's "some tile marked" flag was last read by this step's fused
    // kernel: clear it for step iter+1 to set
    if (blockIdx.x == 0 && threadIdx.x == 0 && d.susp_any) d.susp_any[(iter + 1) & 1] = 0u;
    constexpr int E3 = E * E * E;
    constexpr int G = E + 2;
    __shared__ RouteTab rt;
    __shared__ uint32_t s_solid[(G * G * G + 31) / 32];
    __shared__ int s_tc[3];
    if (d.nactive && d.tile_base + int(blockIdx.x) >= *d.nactive) return;
    const int slot = active[blockIdx.x];
    if (d.no_fluid && d.no_fluid[slot]) return;  // (see Dev::no_fluid)
    const bool marked = d.suspect[slot] != 0;
    if (!marked && !d.screen_all) return;
    if (d.mode[slot] != MODE_PULL) return;  // (every tile that stepped pulls by now)
    const bool hs = d.has_solid[slot] != 0;
    load_routes(rt, d.route[ROUTE_PSI] + size_t(slot) * 18, slot, P.amb_slot, d.slot_f[src_buf]);
    if (threadIdx.x < 3) s_tc[threadIdx.x] = d.coords[slot * 3 + threadIdx.x];
    if (hs)
        for (int k = threadIdx.x; k < d.solid_words; k += NT) s_solid[k] = d.solid[size_t(slot) * d.solid_words + k];
    __syncthreads();
    if (threadIdx.x == 0 && marked) d.suspect[slot] = 0;
    const int tile_lin = (s_tc[0] * P.grid[1] + s_tc[1]) * P.grid[2] + s_tc[2];
    bool bad = false;
    for (int cell = threadIdx.x; cell < E3 && !bad; cell += NT) {
        const int x = cell % E, y = (cell / E) % E, z = cell / (E * E);
        if (hs && solid_at<E>(s_solid, x, y, z)) continue;
#pragma unroll 1
        for (int c = 0; c < C; ++c) {
            double f[Q], rho, u0, u1, u2;
            pull_cell_k<E>(aa_kind(d.aa, iter + 1), rt, c, hs, s_solid, x, y, z, f);
            moments(f, rho, u0, u1, u2);
            if (!isfinite(rho) || !isfinite(u0) || !isfinite(u1) || !isfinite(u2)) bad = true;
        }
    }
    if (bad) atomic_err(d.err, iter, tile_lin, ERR_P5_NAN);
}

// Static batches: after each step, a recorded error halts the steps queued
// behind it (the state then stays at the failing step, as the reference's).
static __global__ void k_err_halt(const unsigned long long* err, int* halt) {
    if (*(volatile const unsigned long long*)err != ERR_NONE_KEY) *halt = 1;
}

// Reference-view read-back of one tile (f_read, rho, u) into out:
// [19*E3 f][E3 rho][E3 ux][E3 uy][E3 uz]
template <int E>
__global__ void k_readback(Dev d, int slot, int c, int src_buf, double* out, int kind) {
    constexpr int E3 = E * E * E;
    constexpr int G = E + 2;
    __shared__ RouteTab rt;
    __shared__ uint32_t s_solid[(G * G * G + 31) / 32];
    __shared__ int s_tc[3];
    const uint8_t mode = d.mode[slot];
    const bool hs = d.has_solid[slot] != 0;
    load_routes(rt, d.route[ROUTE_PULL] + size_t(slot) * 18, slot, P.amb_slot, d.slot_f[src_buf]);
    if (threadIdx.x < 3) s_tc[threadIdx.x] = d.coords[slot * 3 + threadIdx.x];
    if (hs)
        for (int k = threadIdx.x; k < d.solid_words; k += blockDim.x)
            s_solid[k] = d.solid[size_t(slot) * d.solid_words + k];
    __syncthreads();
    for (int cell = blockIdx.x * blockDim.x + threadIdx.x; cell < E3; cell += gridDim.x * blockDim.x) {
        const int x = cell % E, y = (cell / E) % E, z = cell / (E * E);
        double f[Q], u0 = 0.0, u1 = 0.0, u2 = 0.0, rho = 0.0;
        const bool sol = hs && solid_at<E>(s_solid, x, y, z);
        if (sol) {
            for (int i = 0; i < Q; ++i) f[i] = P.comp[c].feq_amb[i];
        } else if (mode == MODE_PULL) {
            pull_cell_k<E>(kind, rt, c, hs, s_solid, x, y, z, f);
            moments(f, rho, u0, u1, u2);
        } else {
            gen_fin<E>(mode, c, s_tc, x, y, z, f, u0, u1, u2);
            // stored density: seed rho / rho_ambient (create_tile + apply_seeds)
            const int s = mode == MODE_GEN_SEEDED ? seed_for<E>(c, s_tc, x, y, z) : -1;
            rho = s >= 0 ? P.seeds[s].rho : P.comp[c].rho_amb;
        }
        for (int i = 0; i < Q; ++i) out[size_t(i) * E3 + cell] = f[i];
        out[size_t(19) * E3 + cell] = rho;
        out[size_t(20) * E3 + cell] = u0;
        out[size_t(21) * E3 + cell] = u1;
        out[size_t(22) * E3 + cell] = u2;
    }
}

// Snapshot gather (dump.cpp:21-57, gather_field): one field of one component
// of every active tile into the domain grid (x fastest), as the reference
// holds it between steps.  kind 0 = rho (0 on solid cells), 1 = |u| =
// sqrt((ux ux + uy uy) + uz uz), 2 = psi (from the capture buffer: psi of the
// step's P1).  grid is pre-filled with the ambient value; grid.y = tile.
template <int E>
__global__ void k_gather(Dev d, const int* __restrict__ active, int kind, int c, int src_buf,
                         double* grid, int D0, int D1, int skind) {
    constexpr int E3 = E * E * E;
    constexpr int G = E + 2;
    __shared__ RouteTab rt;
    __shared__ uint32_t s_solid[(G * G * G + 31) / 32];
    __shared__ int s_tc[3];
    const int slot = active[blockIdx.y];
    const uint8_t mode = d.mode[slot];
    const bool hs = d.has_solid[slot] != 0;
    load_routes(rt, d.route[ROUTE_PULL] + size_t(slot) * 18, slot, P.amb_slot, d.slot_f[src_buf]);
    if (threadIdx.x < 3) s_tc[threadIdx.x] = d.coords[slot * 3 + threadIdx.x];
    if (hs)
        for (int k = threadIdx.x; k < d.solid_words; k += blockDim.x)
            s_solid[k] = d.solid[size_t(slot) * d.solid_words + k];
    __syncthreads();
    const int li = d.lidx[slot];
    for (int cell = blockIdx.x * blockDim.x + threadIdx.x; cell < E3; cell += gridDim.x * blockDim.x) {
        const int x = cell % E, y = (cell / E) % E, z = cell / (E * E);
        const bool sol = hs && solid_at<E>(s_solid, x, y, z);
        double v = 0.0;
        if (kind == 2) {
            v = d.capture[(size_t(li) * P.C + c) * 4 * E3 + cell];
        } else if (!sol || kind == 1) {
            double f[Q], u0 = 0.0, u1 = 0.0, u2 = 0.0, rho = 0.0;
            if (sol) {
                // u of a solid cell is never written by the reference: 0
            } else if (mode == MODE_PULL) {
                pull_cell_k<E>(skind, rt, c, hs, s_solid, x, y, z, f);
                moments(f, rho, u0, u1, u2);
            } else {
                gen_fin<E>(mode, c, s_tc, x, y, z, f, u0, u1, u2);
                const int s = mode == MODE_GEN_SEEDED ? seed_for<E>(c, s_tc, x, y, z) : -1;
                rho = s >= 0 ? P.seeds[s].rho : P.comp[c].rho_amb;
            }
            v = kind == 0 ? rho : sqrt(u0 * u0 + u1 * u1 + u2 * u2);
        }
        grid[size_t(s_tc[0] * E + x) + size_t(D0) * (size_t(s_tc[1] * E + y) + size_t(D1) * size_t(s_tc[2] * E + z))] = v;
    }
}

static __global__ void k_fill(double* p, size_t n, double v) {
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x)
        p[i] = v;
}

// After k_face of a speculatively queued step: does this step's trigger set
// need the host (a birth: an in-bounds absent target), or did an error occur?
// Then set the sticky halt flag and leave the triggers for the host's expand.
// Otherwise count the out-of-bounds triggers as suppressed expansions
// (tilemap.cpp:220-266 counts every out-of-bounds trigger) and clear them, so
// the next queued step proceeds without a host round trip.  One CTA.
static __global__ void k_check(Dev d, const uint8_t* __restrict__ bmask, const uint8_t* __restrict__ omask,
                        int nslot, int* halt) {
    if (*(volatile int*)halt != 0) return;
    __shared__ int s_birth;
    __shared__ unsigned long long s_supp;
    if (threadIdx.x == 0) {
        s_birth = (*d.err != ERR_NONE_KEY) ? 1 : 0;
        s_supp = 0;
    }
    __syncthreads();
    int birth = 0;
    unsigned supp = 0;
    for (int s = threadIdx.x; s < nslot; s += blockDim.x) {
        const unsigned t = d.trig[s];
        birth |= (t & bmask[s]) != 0;
        supp += __popc(t & omask[s]);
    }
    if (__any_sync(0xffffffffu, birth) && (threadIdx.x & 31) == 0) s_birth = 1;
    supp = __reduce_add_sync(0xffffffffu, supp);
    if ((threadIdx.x & 31) == 0 && supp) atomicAdd(&s_supp, (unsigned long long)supp);
    __syncthreads();
    if (s_birth) {
        if (threadIdx.x == 0) *halt = 1;
        return;
    }
    for (int s = threadIdx.x; s < nslot; s += blockDim.x) d.trig[s] = 0;
    if (threadIdx.x == 0 && s_supp) d.cnt[CNT_SUPP] += s_supp;
}

}  // namespace plbm
