// kernels_tm.cuh — k_main_tm: the default fused step kernel (sm_100a).
//
// Why not a plain stencil: the Shan-Chen force needs psi of all 18
// neighbours, and psi needs the density of the POST-STREAM populations, so
// each cell's pulled f_in is used twice — once for rho -> psi (one plane
// ahead), once for the collision.  Pulling twice misses L2 (reuse distance
// ~90 MB chip-wide; ncu: DRAM reads 2.4x the algorithmic bytes), so the first
// pull is the only one and its 19*C doubles stay on chip until the collide:
//   * even planes in Tensor Memory (tcgen05.st / tcgen05.ld, 32x32b shape,
//     one TMEM lane per thread) — 256 KB per SM this FP64 stencil otherwise
//     never uses;
//   * odd planes in shared memory;
// which lets two CTAs (16 warps) share an SM at <= 128 registers per thread.
//
// Decomposition: one CTA = a 32 x 8 (x, y) column block of one 32^3 tile,
// marching z over the whole tile; the four blocks of a tile form a thread-
// block cluster.  Block rows 0 and BY-1 push their psi values straight into
// the neighbouring block's shared ring with st.async, completing transactions
// on the receiver's mbarrier — no per-plane cluster barrier, no GPU-scope
// fence.  Halo planes / rows outside the tile come from the neighbours' psi
// faces (k_face) through the ghost routing table.
//
// Per plane z:  psi pass of plane z+1 (pull, rho, psi, stash, push rows)
//               | CTA barrier | edge rows wait on the mbarrier | collide z.
#pragma once

#include "kernels.cuh"

namespace plbm {

template <int E, int C>
struct TmCfg {
    static constexpr int NT = 256;
    static constexpr int BY = NT / E;            // rows per CTA
    static constexpr int NB = E / BY;            // CTAs per tile = cluster size
    static constexpr int CB = 40;                // TMEM columns per component (38 used)
    static constexpr int NCOLS = 256;            // per CTA; two CTAs per SM
    static constexpr int HALF = NCOLS / 2;       // per warp (two warps per lane quarter)
    static constexpr int PW = E + 2;             // psi plane row pitch (x + ring)
    static constexpr int PH = BY + 2;
    static constexpr int PP = PW * PH;
    static constexpr int PSI_BYTES = 4 * C * PP * 8;
    static constexpr int STAGE_BYTES = Q * C * NT * 8;
    static constexpr int SMEM = PSI_BYTES + STAGE_BYTES;
    static_assert(CB * C <= HALF, "TMEM slot does not fit");
    static_assert(2 * (SMEM + 6 * 1024) <= 228 * 1024, "two CTAs per SM must fit");
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// 19 doubles = 38 TMEM columns of this thread's lane, written as 32x32b
// x8,x8,x8,x8,x4,x2 chunks at offsets aligned to the chunk width (each
// component block starts on an 8-column boundary: CB = 40 columns).
#define PLBM_TM_ST8(A, R, o)                                                                     \
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};\n" \
                 ::"r"(A), "r"(R[o]), "r"(R[o + 1]), "r"(R[o + 2]), "r"(R[o + 3]), "r"(R[o + 4]), \
                 "r"(R[o + 5]), "r"(R[o + 6]), "r"(R[o + 7]))
#define PLBM_TM_LD8(A, R, o)                                                                     \
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];\n" \
                 : "=r"(R[o]), "=r"(R[o + 1]), "=r"(R[o + 2]), "=r"(R[o + 3]), "=r"(R[o + 4]),    \
                   "=r"(R[o + 5]), "=r"(R[o + 6]), "=r"(R[o + 7])                                 \
                 : "r"(A))

__device__ __forceinline__ void tm_store19(uint32_t taddr, const double* f) {
    uint32_t r[38];
#pragma unroll
    for (int i = 0; i < 19; ++i) {
        r[2 * i] = uint32_t(__double2loint(f[i]));
        r[2 * i + 1] = uint32_t(__double2hiint(f[i]));
    }
    PLBM_TM_ST8(taddr, r, 0);
    PLBM_TM_ST8(taddr + 8, r, 8);
    PLBM_TM_ST8(taddr + 16, r, 16);
    PLBM_TM_ST8(taddr + 24, r, 24);
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};\n" ::"r"(taddr + 32),
                 "r"(r[32]), "r"(r[33]), "r"(r[34]), "r"(r[35]));
    asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1, %2};\n" ::"r"(taddr + 36),
                 "r"(r[36]), "r"(r[37]));
}

__device__ __forceinline__ void tm_load19(uint32_t taddr, double* f) {
    uint32_t r[38];
    PLBM_TM_LD8(taddr, r, 0);
    PLBM_TM_LD8(taddr + 8, r, 8);
    PLBM_TM_LD8(taddr + 16, r, 16);
    PLBM_TM_LD8(taddr + 24, r, 24);
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];\n"
                 : "=r"(r[32]), "=r"(r[33]), "=r"(r[34]), "=r"(r[35])
                 : "r"(taddr + 32));
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0, %1}, [%2];\n"
                 : "=r"(r[36]), "=r"(r[37])
                 : "r"(taddr + 36));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
    for (int i = 0; i < 19; ++i) f[i] = __hiloint2double(int(r[2 * i + 1]), int(r[2 * i]));
}

// One component's collision at one cell (engine.cpp:420-476): gravity +
// intra + inter force, then BGK with the velocity-shift forcing.  pm0/p00/pp0
// point at this cell's psi in planes z-1, z, z+1 for component 0; component k
// is CP doubles further.
template <int C, int PW, int CP>
__device__ __forceinline__ void collide_comp(const double* f, double rho, double u0, double u1,
                                             double u2, int c, const double* pm0,
                                             const double* p00, const double* pp0,
                                             double* out, size_t dstride, int& zero_rho) {
    const double* pm_c = pm0 + c * CP;
    const double* p0_c = p00 + c * CP;
    const double* pp_c = pp0 + c * CP;
    const CompConst& kc = P.comp[c];
    double F0 = 0.0, F1 = 0.0, F2 = 0.0;
    if (kc.has_gravity) {
        F0 = rho * kc.gravity[0];
        F1 = rho * kc.gravity[1];
        F2 = rho * kc.gravity[2];
    }
    {  // intra_force, proj/src/physics.cpp:44-63
        double s10 = 0.0, s11 = 0.0, s12 = 0.0, s20 = 0.0, s21 = 0.0, s22 = 0.0;
#pragma unroll
        for (int i = 1; i < Q; ++i) {
            const int dx = ex_(i), dy = ey_(i), dz = ez_(i);
            const double* pl = dz < 0 ? pm_c : (dz > 0 ? pp_c : p0_c);
            const double pn = pl[dx + PW * dy];
            const double a1 = w_(i) * pn;
            const double a2 = a1 * pn;
            if (dx > 0) { s10 += a1; s20 += a2; }
            if (dx < 0) { s10 -= a1; s20 -= a2; }
            if (dy > 0) { s11 += a1; s21 += a2; }
            if (dy < 0) { s11 -= a1; s21 -= a2; }
            if (dz > 0) { s12 += a1; s22 += a2; }
            if (dz < 0) { s12 -= a1; s22 -= a2; }
        }
        const double c1 = kc.c1f * p0_c[0];
        const double c2 = kc.c2;
        F0 += c1 * s10 + c2 * s20;
        F1 += c1 * s11 + c2 * s21;
        F2 += c1 * s12 + c2 * s22;
    }
#pragma unroll
    for (int c2i = 0; c2i < C; ++c2i) {  // inter_force, proj/src/physics.cpp:65-78
        if (c2i == c) continue;
        const double g = P.coupling[c * C + c2i];
        if (g == 0.0) continue;
        double t0 = 0.0, t1 = 0.0, t2 = 0.0;
#pragma unroll
        for (int i = 1; i < Q; ++i) {
            const int dx = ex_(i), dy = ey_(i), dz = ez_(i);
            const double* pl = (dz < 0 ? pm0 : (dz > 0 ? pp0 : p00)) + c2i * CP;
            const double a1 = w_(i) * pl[dx + PW * dy];
            if (dx > 0) t0 += a1;
            if (dx < 0) t0 -= a1;
            if (dy > 0) t1 += a1;
            if (dy < 0) t1 -= a1;
            if (dz > 0) t2 += a1;
            if (dz < 0) t2 -= a1;
        }
        const double cc = (-g) * p0_c[0];
        F0 += cc * t0;
        F1 += cc * t1;
        F2 += cc * t2;
    }
    // ---- collision (engine.cpp:450-475)
    const double om = kc.omega;
    const double uu = u0 * u0 + u1 * u1 + u2 * u2;
    const double t3 = (0.5 * uu) * 3.0;
    const double wr0 = PLBM_W0 * rho, wr1 = PLBM_W1 * rho, wr2 = PLBM_W2 * rho;
    const bool unforced = (F0 == 0.0 && F1 == 0.0 && F2 == 0.0);
    if (!unforced && rho <= 0.0) ++zero_rho;
    if (unforced || rho <= 0.0) {
#define PLBM_TM_RELAX(I)                                                                      \
    {                                                                                         \
        constexpr int IP = (I == 0 ? 1 : I - ((I + 1) & 1));                                  \
        const double wr = (I == 0) ? wr0 : ((I <= 6) ? wr1 : wr2);                            \
        const double eu = (I == 0) ? 0.0 : eu_pair<IP>(u0, u1, u2);                           \
        const double e0 = feq_dir<I>(wr, eu, t3);                                             \
        out[size_t(I) * dstride] = f[I] + om * (e0 - f[I]);                                   \
    }
        PLBM_TM_RELAX(0) PLBM_TM_RELAX(1) PLBM_TM_RELAX(2) PLBM_TM_RELAX(3) PLBM_TM_RELAX(4)
        PLBM_TM_RELAX(5) PLBM_TM_RELAX(6) PLBM_TM_RELAX(7) PLBM_TM_RELAX(8) PLBM_TM_RELAX(9)
        PLBM_TM_RELAX(10) PLBM_TM_RELAX(11) PLBM_TM_RELAX(12) PLBM_TM_RELAX(13) PLBM_TM_RELAX(14)
        PLBM_TM_RELAX(15) PLBM_TM_RELAX(16) PLBM_TM_RELAX(17) PLBM_TM_RELAX(18)
#undef PLBM_TM_RELAX
    } else {
        const double v0 = u0 + F0 / rho, v1 = u1 + F1 / rho, v2 = u2 + F2 / rho;
        const double vv = v0 * v0 + v1 * v1 + v2 * v2;
        const double s3 = (0.5 * vv) * 3.0;
#define PLBM_TM_FORCED(I)                                                                     \
    {                                                                                         \
        constexpr int IP = (I == 0 ? 1 : I - ((I + 1) & 1));                                  \
        const double wr = (I == 0) ? wr0 : ((I <= 6) ? wr1 : wr2);                            \
        const double eu = (I == 0) ? 0.0 : eu_pair<IP>(u0, u1, u2);                           \
        const double ev = (I == 0) ? 0.0 : eu_pair<IP>(v0, v1, v2);                           \
        const double e0 = feq_dir<I>(wr, eu, t3);                                             \
        const double e1 = feq_dir<I>(wr, ev, s3);                                             \
        out[size_t(I) * dstride] = f[I] + ((om * (e0 - f[I]) + e1) - e0);                     \
    }
        PLBM_TM_FORCED(0) PLBM_TM_FORCED(1) PLBM_TM_FORCED(2) PLBM_TM_FORCED(3)
        PLBM_TM_FORCED(4) PLBM_TM_FORCED(5) PLBM_TM_FORCED(6) PLBM_TM_FORCED(7)
        PLBM_TM_FORCED(8) PLBM_TM_FORCED(9) PLBM_TM_FORCED(10) PLBM_TM_FORCED(11)
        PLBM_TM_FORCED(12) PLBM_TM_FORCED(13) PLBM_TM_FORCED(14) PLBM_TM_FORCED(15)
        PLBM_TM_FORCED(16) PLBM_TM_FORCED(17) PLBM_TM_FORCED(18)
#undef PLBM_TM_FORCED
    }
}

// Seed / ambient velocity of a GEN-mode cell (the u the reference holds
// before a tile's first collision).
template <int E>
__device__ __forceinline__ void gen_u(int mode, int c, const int* tc, int x, int y, int z,
                                      double& u0, double& u1, double& u2) {
    const int s = (mode == MODE_GEN_SEEDED) ? seed_for<E>(c, tc, x, y, z) : -1;
    if (s >= 0) {
        u0 = P.seeds[s].u[0];
        u1 = P.seeds[s].u[1];
        u2 = P.seeds[s].u[2];
    } else {
        u0 = u1 = u2 = 0.0;
    }
}

template <int E, int C>
__global__ void __launch_bounds__(256, 2) k_main_tm(Dev d, const int* __restrict__ active,
                                                    int src_buf, int write_uface, long iter) {
    using T = TmCfg<E, C>;
    constexpr int NT = T::NT, BY = T::BY, NB = T::NB, PW = T::PW, PH = T::PH, PP = T::PP;
    constexpr int G = E + 2;
    constexpr int E2 = E * E;
    constexpr int E3 = E * E * E;
    static_assert(NB == 1 || BY * E == NT, "one warp per block row");
    extern __shared__ __align__(16) double smem[];
    double* psi = smem;                 // [4][C][PH][PW] ring of psi planes
    double* stage = smem + 4 * C * PP;  // [C][Q][NT] odd-plane stash
    __shared__ RouteTab rt_pull, rt_psi;
    __shared__ uint32_t s_solid[(G * G * G + 31) / 32];
    __shared__ int s_tc[3];
    __shared__ uint32_t s_tmem;
    __shared__ __align__(8) uint64_t s_mbar[2];  // psi-row arrival, by plane parity

    const int tid = threadIdx.x;
    const int warp = tid >> 5;
    const int tile_i = blockIdx.x / NB;
    const int yb = blockIdx.x % NB;
    const int y0 = yb * BY;
    const int slot = active[tile_i];
    const uint8_t mode = d.mode[slot];
    const bool hs = d.has_solid[slot] != 0;
    const int amb = P.amb_slot;
    const int par = int(iter & 1);
    double* __restrict__ fo = d.slot_f[src_buf ^ 1][slot];
    const int li = d.lidx[slot];

    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                         smem_u32(&s_tmem)),
                     "n"(T::NCOLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    load_routes(rt_pull, d.route[ROUTE_PULL] + size_t(slot) * 18, slot, amb, d.slot_f[src_buf]);
    load_routes(rt_psi, d.route[ROUTE_PSI] + size_t(slot) * 18, slot, amb, d.slot_pf[par], d.mode);
    if (tid < 3) s_tc[tid] = d.coords[slot * 3 + tid];
    if (hs)
        for (int k = tid; k < d.solid_words; k += NT) s_solid[k] = d.solid[size_t(slot) * d.solid_words + k];
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(&s_mbar[0])), "r"(1));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(&s_mbar[1])), "r"(1));
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    // peers must see our initialised mbarriers before they push rows at us
    if constexpr (NB > 1) {
        asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
        asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
    }
    const uint32_t tbase = s_tmem + (uint32_t(32 * (warp & 3)) << 16) + uint32_t((warp >> 2) * T::HALF);
    const int tile_lin = (s_tc[0] * P.grid[1] + s_tc[1]) * P.grid[2] + s_tc[2];

    const int x = tid % E;
    const int yl = tid / E;
    const int y = y0 + yl;
    // fast pull applies to this warp's row(s): no solids, y+-1 inside the tile
    // (E = 32: one warp is one row, so the test is warp-uniform)
    const bool fast_rows = mode == MODE_PULL && !hs && y >= 1 && y <= E - 2;
    auto pidx = [&](int ring, int c, int xx, int yy_local) {
        return ((ring * C + c) * PH + (yy_local + 1)) * PW + (xx + 1);
    };

    // ---- push-based psi row exchange --------------------------------------
    // Block row 0 feeds the -y neighbour's ring row BY, block row BY-1 feeds
    // the +y neighbour's ring row -1: each value goes out as an 8-byte st.async
    // that completes a transaction on the receiver's mbarrier.
    const bool push_lo = NB > 1 && yl == 0 && yb > 0;
    const bool push_hi = NB > 1 && yl == BY - 1 && yb < NB - 1;
    uint32_t peer_psi = 0, peer_mbar = 0;
    if (push_lo || push_hi) {
        const uint32_t nb = uint32_t(yb + (push_lo ? -1 : 1));
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(peer_psi) : "r"(smem_u32(psi)), "r"(nb));
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n"
                     : "=r"(peer_mbar)
                     : "r"(smem_u32(&s_mbar[0])), "r"(nb));
    }
    const uint32_t rows_bytes = uint32_t(((yb > 0) + (yb < NB - 1)) * E * C * 8);
    auto push_row = [&](int pz, int c, double v) {
        if (!(push_lo || push_hi)) return;
        const int idx = pidx(pz & 3, c, x, push_lo ? BY : -1);
        asm volatile(
            "st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];\n" ::"r"(
                peer_psi + uint32_t(idx) * 8u),
            "l"(__double_as_longlong(v)), "r"(peer_mbar + uint32_t((pz & 1) * 8))
            : "memory");
    };
    auto expect_rows = [&](int pz) {
        if (NB > 1 && tid == 0)
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(
                             smem_u32(&s_mbar[pz & 1])),
                         "r"(rows_bytes)
                         : "memory");
    };
    // only the rows that read a pushed ring row wait for it
    const bool needs_rows = NB > 1 && ((yl == 0 && yb > 0) || (yl == BY - 1 && yb < NB - 1));
    auto wait_rows = [&](int pz) {
        if (!needs_rows) return;
        const uint32_t bar = smem_u32(&s_mbar[pz & 1]);
        const uint32_t parity = uint32_t((pz >> 1) & 1);
        uint32_t ok = 0;
        while (!ok)
            asm volatile(
                "{\n .reg .pred q;\n mbarrier.try_wait.parity.shared::cta.b64 q, [%1], %2;\n"
                " selp.u32 %0, 1, 0, q;\n}\n"
                : "=r"(ok)
                : "r"(bar), "r"(parity)
                : "memory");
    };

    // ---- psi of out-of-block positions (face buffers of neighbour tiles) ----
    auto fill_zghost = [&](int pz) {  // whole plane outside the tile in z
        const int ring = pz & 3;
        for (int k = tid; k < PP; k += NT) {
            const int xx = k % PW - 1, yy = k / PW - 1 + y0;
            const bool xo = xx < 0 || xx >= E, yo = yy < 0 || yy >= E;
#pragma unroll 1
            for (int c = 0; c < C; ++c)
                psi[pidx(ring, c, xx, yy - y0)] =
                    (xo && yo) ? 0.0 : psi_ghost<E>(rt_psi, c, hs, s_solid, xx, yy, pz);
        }
    };
    auto fill_ring = [&](int pz) {  // x ring + y rows that lie outside the tile
        const int ring = pz & 3;
        for (int k = tid; k < 2 * PH + 2 * E; k += NT) {
            int xx, yyl;
            if (k < 2 * PH) {
                xx = (k & 1) ? E : -1;
                yyl = (k >> 1) - 1;
            } else {
                const int q = k - 2 * PH;
                xx = q % E;
                yyl = (q / E) ? BY : -1;
                const int yy = y0 + yyl;
                if (yy >= 0 && yy < E) continue;  // pushed by the cluster neighbour
            }
#pragma unroll 1
            for (int c = 0; c < C; ++c)
                psi[pidx(ring, c, xx, yyl)] = psi_ghost<E>(rt_psi, c, hs, s_solid, xx, y0 + yyl, pz);
        }
    };

    // ---- psi pass of plane pz: pull f_in, rho -> psi (P1), stash -------------
    auto psi_pass = [&](int pz) {
        const int ring = pz & 3;
        const bool sol = hs && solid_at<E>(s_solid, x, y, pz);
        int negs = 0, clamps = 0;
#pragma unroll 1
        for (int c = 0; c < C; ++c) {
            double f[Q];
            double v = 0.0;
            if (sol) {
#pragma unroll
                for (int i = 0; i < Q; ++i) f[i] = 0.0;
            } else {
                if (fast_rows && pz >= 1 && pz <= E - 2) {
                    pull_cell_fast<E>(rt_pull, c, x, y, pz, f);
                } else if (mode == MODE_PULL) {
                    pull_cell<E>(rt_pull, c, hs, s_solid, x, y, pz, f);
                } else {
                    double a0, a1, a2;
                    gen_fin<E>(mode, c, s_tc, x, y, pz, f, a0, a1, a2);
                }
                double rho = 0.0;
#pragma unroll
                for (int i = 0; i < Q; ++i) {
                    rho += f[i];
                    negs += f[i] < 0.0;
                }
                if (!isfinite(rho)) {
                    atomic_err(d.err, iter, tile_lin, ERR_P1_NAN);
                } else {
                    double press;
                    if (!pr_pressure(rho, P.comp[c], press)) {
                        atomic_err(d.err, iter, tile_lin, ERR_P1_POLE);
                    } else {
                        bool cl;
                        v = pseudo_potential(rho, press, P.comp[c], cl);
                        clamps += cl;
                    }
                }
            }
            psi[pidx(ring, c, x, yl)] = v;
            push_row(pz, c, v);
            if ((pz & 1) == 0) {
                tm_store19(tbase + uint32_t(c * T::CB), f);
            } else {
                double* st = stage + size_t(c) * Q * NT + tid;
#pragma unroll
                for (int i = 0; i < Q; ++i) st[i * NT] = f[i];
            }
        }
        if ((pz & 1) == 0) asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
        const unsigned m1 = __reduce_add_sync(0xffffffffu, (unsigned)negs);
        const unsigned m2 = __reduce_add_sync(0xffffffffu, (unsigned)clamps);
        if ((tid & 31) == 0) {
            if (m1) atomicAdd(&d.cnt[CNT_NEG], (unsigned long long)m1);
            if (m2) atomicAdd(&d.cnt[CNT_CLAMP], (unsigned long long)m2);
        }
    };

    // ---- collide plane z from its stash ---------------------------------------
    auto collide_plane = [&](int z) {
        const bool sol = hs && solid_at<E>(s_solid, x, y, z);
        const int cell = (z * E + y) * E + x;
        const double* pm = psi + pidx((z - 1) & 3, 0, x, yl);
        const double* p0 = psi + pidx(z & 3, 0, x, yl);
        const double* ppl = psi + pidx((z + 1) & 3, 0, x, yl);
        unsigned fmask = 0;  // frontier faces this cell lies on (criterion u_prev)
        if (write_uface) {
#pragma unroll
            for (int face = 0; face < 6; ++face) {
                const int axis = face >> 1;
                const int coord = axis == 0 ? x : (axis == 1 ? y : z);
                if (coord == ((face & 1) ? E - 1 : 0) && rt_psi.s[face_pattern(face)] == amb)
                    fmask |= 1u << face;
            }
        }
        int zero_rho = 0;
#pragma unroll 1
        for (int c = 0; c < C; ++c) {
            double f[Q];
            if ((z & 1) == 0) {
                tm_load19(tbase + uint32_t(c * T::CB), f);  // warp-convergent
            } else {
                const double* st = stage + size_t(c) * Q * NT + tid;
#pragma unroll
                for (int i = 0; i < Q; ++i) f[i] = st[i * NT];
            }
            if (sol) continue;
            double rho, u0 = 0.0, u1 = 0.0, u2 = 0.0;
            if (mode == MODE_PULL) {
                moments(f, rho, u0, u1, u2);
            } else {
                rho = sum19(f);
                gen_u<E>(mode, c, s_tc, x, y, z, u0, u1, u2);
            }
            if (fmask) {
#pragma unroll 1
                for (int face = 0; face < 6; ++face) {
                    if (!(fmask & (1u << face))) continue;
                    double* uf = d.u_face + ((size_t(li) * C + c) * 6 + face) * 3 * E2;
                    const int fi = face_index<E>(face, x, y, z);
                    uf[fi] = u0;
                    uf[E2 + fi] = u1;
                    uf[2 * E2 + fi] = u2;
                }
            }
            if (d.capture) {
                double* cp = d.capture + (size_t(li) * C + c) * 4 * E3;
                cp[cell] = p0[c * PP];
                cp[E3 + cell] = u0;
                cp[2 * E3 + cell] = u1;
                cp[3 * E3 + cell] = u2;
            }
            double* out = fo + c * size_t(Q) * E3 + cell;
            collide_comp<C, PW, PP>(f, rho, u0, u1, u2, c, pm, p0, ppl, out, size_t(E3), zero_rho);
        }
        const unsigned zr = __reduce_add_sync(0xffffffffu, (unsigned)zero_rho);
        if ((tid & 31) == 0 && zr) atomicAdd(&d.cnt[CNT_ZERO_RHO], (unsigned long long)zr);
    };

    fill_zghost(-1);
    expect_rows(0);
    psi_pass(0);
    fill_ring(0);
    __syncthreads();
    wait_rows(0);
#pragma unroll 1
    for (int z = 0; z < E; ++z) {
        if (z + 1 < E) {
            expect_rows(z + 1);
            psi_pass(z + 1);
            fill_ring(z + 1);
        } else {
            fill_zghost(E);
        }
        __syncthreads();
        if (z + 1 < E) wait_rows(z + 1);
        collide_plane(z);
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    if constexpr (NB > 1) {  // all pushes into peers have landed before anyone exits
        asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
        asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
    }
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(s_tmem),
                     "n"(T::NCOLS));
}

}  // namespace plbm
