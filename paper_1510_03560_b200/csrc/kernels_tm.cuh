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
    static constexpr int CB = 40;                // TMEM columns per component: 19 f + rho
    static constexpr int NCOLS = 256;            // per CTA; two CTAs per SM
    static constexpr int HALF = NCOLS / 2;       // per warp (two warps per lane quarter)
    static constexpr int PW = E + 2;             // psi plane row pitch (x + ring)
    static constexpr int PH = BY + 2;
    static constexpr int PP = PW * PH;
    static constexpr int PSI_BYTES = 4 * C * PP * 8;
    static constexpr int STAGE_BYTES = (Q + 1) * C * NT * 8;  // 19 f + rho
    static constexpr int SMEM = PSI_BYTES + STAGE_BYTES;
    static_assert(CB * C <= HALF, "TMEM slot does not fit");
    static_assert(2 * (SMEM + 6 * 1024) <= 228 * 1024, "two CTAs per SM must fit");
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// 19 populations + rho = 40 TMEM columns of this thread's lane, written as
// one 32x32b.x32 and one .x8 chunk (each component block starts on an
// 8-column boundary: CB = 40 columns).
__device__ __forceinline__ void tm_store20(uint32_t taddr, const double* f, double rho) {
    uint32_t r[40];
#pragma unroll
    for (int i = 0; i < 19; ++i) {
        r[2 * i] = uint32_t(__double2loint(f[i]));
        r[2 * i + 1] = uint32_t(__double2hiint(f[i]));
    }
    r[38] = uint32_t(__double2loint(rho));
    r[39] = uint32_t(__double2hiint(rho));
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
        "%11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, "
        "%29, %30, %31, %32};\n" ::"r"(taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
        "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]),
        "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]),
        "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31]));
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};\n" ::"r"(
                     taddr + 32),
                 "r"(r[32]), "r"(r[33]), "r"(r[34]), "r"(r[35]), "r"(r[36]), "r"(r[37]), "r"(r[38]),
                 "r"(r[39]));
}

__device__ __forceinline__ void tm_load20(uint32_t taddr, double* f, double& rho) {
    uint32_t r[40];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, "
        "%12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, "
        "%30, %31}, [%32];\n"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
          "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]),
          "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]),
          "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];\n"
                 : "=r"(r[32]), "=r"(r[33]), "=r"(r[34]), "=r"(r[35]), "=r"(r[36]), "=r"(r[37]),
                   "=r"(r[38]), "=r"(r[39])
                 : "r"(taddr + 32));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
    for (int i = 0; i < 19; ++i) f[i] = __hiloint2double(int(r[2 * i + 1]), int(r[2 * i]));
    rho = __hiloint2double(int(r[39]), int(r[38]));
}

// Shan-Chen sums of component k over the 18 neighbours (physics.cpp:44-78):
// s1 = sum (w psi_n) e_i, s2 = sum ((w psi_n) psi_n) e_i, in i order with the
// zero-e terms folded.  inter_force's sum for (c <- k) is the same expression
// in the same order as intra_force's s1 of k, so it is computed once per k and
// shared (bit-identical).  pl[dz+1] points at this cell's psi of component k
// in planes z-1, z, z+1.
template <int PW, bool S2>
__device__ __forceinline__ void sc_sums(const double* pm, const double* p0, const double* pp,
                                        double* s1, double* s2) {
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, b0 = 0.0, b1 = 0.0, b2 = 0.0;
#pragma unroll
    for (int i = 1; i < Q; ++i) {
        const int dx = ex_(i), dy = ey_(i), dz = ez_(i);
        const double* pl = dz < 0 ? pm : (dz > 0 ? pp : p0);
        const double pn = pl[dx + PW * dy];
        const double t1 = w_(i) * pn;
        if (dx > 0) a0 += t1;
        if (dx < 0) a0 -= t1;
        if (dy > 0) a1 += t1;
        if (dy < 0) a1 -= t1;
        if (dz > 0) a2 += t1;
        if (dz < 0) a2 -= t1;
        if constexpr (S2) {
            const double t2 = t1 * pn;
            if (dx > 0) b0 += t2;
            if (dx < 0) b0 -= t2;
            if (dy > 0) b1 += t2;
            if (dy < 0) b1 -= t2;
            if (dz > 0) b2 += t2;
            if (dz < 0) b2 -= t2;
        }
    }
    s1[0] = a0; s1[1] = a1; s1[2] = a2;
    if constexpr (S2) { s2[0] = b0; s2[1] = b1; s2[2] = b2; }
}

// Force of every component at one cell, without gravity (engine.cpp:420-449):
// Fi[c] = intra_force, Fx[c] = the inter_force term (C <= 2: at most one).  Gravity
// (the first term of the reference's sum) is added by the caller, so the
// accumulation order stays ((rho g + Fi) + Fx_c2...).
template <int C, int PW, int CP>
__device__ __forceinline__ void forces_all(const double* pm0, const double* p00, const double* pp0,
                                           double (&Fi)[C][3], double (&Fx)[C][3], bool (&has_x)[C]) {
    static_assert(C <= 2, "k_main_tm handles one or two components");
    double s1[C][3];
#pragma unroll
    for (int k = 0; k < C; ++k) {
        double s2[3];
        sc_sums<PW, true>(pm0 + k * CP, p00 + k * CP, pp0 + k * CP, s1[k], s2);
        const double c1 = P.comp[k].c1f * p00[k * CP];
        const double c2 = P.comp[k].c2;
#pragma unroll
        for (int a = 0; a < 3; ++a) Fi[k][a] = c1 * s1[k][a] + c2 * s2[a];
    }
    // C <= 2: at most one coupling term per component
#pragma unroll
    for (int c = 0; c < C; ++c) {
        has_x[c] = false;
        Fx[c][0] = Fx[c][1] = Fx[c][2] = 0.0;
        if constexpr (C == 2) {
            const int k = 1 - c;
            const double g = P.coupling[c * C + k];
            if (g != 0.0) {
                const double cc = (-g) * p00[c * CP];
#pragma unroll
                for (int a = 0; a < 3; ++a) Fx[c][a] = cc * s1[k][a];
                has_x[c] = true;
            }
        }
    }
}

// One component's BGK collision with the velocity-shift forcing
// (engine.cpp:450-475) given the total force F.  f is overwritten with the
// post-collision populations; xc (x-column lanes only, else nullptr) receives
// a copy of all 19 at stride xstride.
__device__ __forceinline__ void collide_bgk(double* f, double rho, double u0, double u1,
                                            double u2, double F0, double F1, double F2,
                                            double om, double* out, size_t dstride,
                                            int& zero_rho, double* xc = nullptr, int xstride = 0) {

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
        f[I] = f[I] + om * (e0 - f[I]);                                                       \
        out[size_t(I) * dstride] = f[I];                                                      \
    }
        PLBM_TM_RELAX(0) PLBM_TM_RELAX(1) PLBM_TM_RELAX(2) PLBM_TM_RELAX(3) PLBM_TM_RELAX(4)
        PLBM_TM_RELAX(5) PLBM_TM_RELAX(6) PLBM_TM_RELAX(7) PLBM_TM_RELAX(8) PLBM_TM_RELAX(9)
        PLBM_TM_RELAX(10) PLBM_TM_RELAX(11) PLBM_TM_RELAX(12) PLBM_TM_RELAX(13) PLBM_TM_RELAX(14)
        PLBM_TM_RELAX(15) PLBM_TM_RELAX(16) PLBM_TM_RELAX(17) PLBM_TM_RELAX(18)
#undef PLBM_TM_RELAX
    } else {
        bool ok = true;
        const double rr = rcp_nv(rho);
        double q0 = div_nv(F0, rho, rr, ok), q1 = div_nv(F1, rho, rr, ok), q2 = div_nv(F2, rho, rr, ok);
        if (!ok) {
            q0 = F0 / rho;
            q1 = F1 / rho;
            q2 = F2 / rho;
        }
        const double v0 = u0 + q0, v1 = u1 + q1, v2 = u2 + q2;
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
        f[I] = f[I] + ((om * (e0 - f[I]) + e1) - e0);                                         \
        out[size_t(I) * dstride] = f[I];                                                      \
    }
        PLBM_TM_FORCED(0) PLBM_TM_FORCED(1) PLBM_TM_FORCED(2) PLBM_TM_FORCED(3)
        PLBM_TM_FORCED(4) PLBM_TM_FORCED(5) PLBM_TM_FORCED(6) PLBM_TM_FORCED(7)
        PLBM_TM_FORCED(8) PLBM_TM_FORCED(9) PLBM_TM_FORCED(10) PLBM_TM_FORCED(11)
        PLBM_TM_FORCED(12) PLBM_TM_FORCED(13) PLBM_TM_FORCED(14) PLBM_TM_FORCED(15)
        PLBM_TM_FORCED(16) PLBM_TM_FORCED(17) PLBM_TM_FORCED(18)
#undef PLBM_TM_FORCED
    }
    // x-column lanes: all 19 post-collision values to the staging area
    if (xc) {
#pragma unroll
        for (int i = 0; i < Q; ++i) xc[i * xstride] = f[i];
    }
}

// Momentum by sequential sums (kernels.hpp:31-48) and u = m / rho, with rho
// the P1 density of the same populations (same sum, same order).
__device__ __forceinline__ void velocity(const double* f, double r, double& u0, double& u1,
                                         double& u2) {
    double m0 = 0.0;
    m0 += f[1]; m0 -= f[2]; m0 += f[7]; m0 -= f[8]; m0 += f[9]; m0 -= f[10];
    m0 += f[11]; m0 -= f[12]; m0 += f[13]; m0 -= f[14];
    double m1 = 0.0;
    m1 += f[3]; m1 -= f[4]; m1 += f[7]; m1 -= f[8]; m1 -= f[9]; m1 += f[10];
    m1 += f[15]; m1 -= f[16]; m1 += f[17]; m1 -= f[18];
    double m2 = 0.0;
    m2 += f[5]; m2 -= f[6]; m2 += f[11]; m2 -= f[12]; m2 -= f[13]; m2 += f[14];
    m2 += f[15]; m2 -= f[16]; m2 -= f[17]; m2 += f[18];
    if (r != 0.0) {
        bool ok = true;
        const double rr = rcp_nv(r);
        u0 = div_nv(m0, r, rr, ok);
        u1 = div_nv(m1, r, rr, ok);
        u2 = div_nv(m2, r, rr, ok);
        if (!ok) {
            u0 = m0 / r;
            u1 = m1 / r;
            u2 = m2 / r;
        }
    } else {
        u0 = u1 = u2 = 0.0;
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

// OPT bits (A/B variants, all bit-identical)
// (Measured and removed: both components' loads in flight together, an L2
// bulk prefetch of the next plane, per-warp mbarrier sync instead of the CTA
// barrier — none faster.)
constexpr int TM_MEMONLY = 8; // measurement only (NOT the physics): same loads, stash and stores, no FP64 work
constexpr int TM_DEFAULT_OPT = 0;

template <int E, int C, int OPT>
__global__ void __launch_bounds__(256, 2) k_main_tm(Dev d, const int* __restrict__ active,
                                                    int src_buf, int write_uface, long iter) {
    if (halted(d)) return;
    using T = TmCfg<E, C>;
    constexpr int NT = T::NT, BY = T::BY, NB = T::NB, PW = T::PW, PH = T::PH, PP = T::PP;
    constexpr int G = E + 2;
    constexpr int E2 = E * E;
    constexpr int E3 = E * E * E;
    static_assert(NB == 1 || BY * E == NT, "one warp per block row");
    extern __shared__ __align__(16) double smem[];
    double* psi = smem;                 // [4][C][PH][PW] ring of psi planes
    double* stage = smem + 4 * C * PP;  // [C][Q+1][NT] odd-plane stash (19 f + rho)
    __shared__ RouteTab rt_pull, rt_psi;
    __shared__ uint32_t s_solid[(G * G * G + 31) / 32];
    __shared__ int s_tc[3];
    __shared__ uint32_t s_tmem;
    // pushed psi rows by plane parity: [0..1] row -1 (from the -y peer, read by
    // block row 0), [2..3] row BY (from the +y peer, read by block row BY-1)
    __shared__ __align__(8) uint64_t s_mbar[4];

    const int tid = threadIdx.x;
    const int warp = tid >> 5;
    const int tile_i = blockIdx.x / NB;
    const int yb = blockIdx.x % NB;
    const int y0 = yb * BY;
    if (d.nactive && d.tile_base + tile_i >= *d.nactive) return;  // (whole clusters: same tile)
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
        for (int k = 0; k < 4; ++k)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(&s_mbar[k])), "r"(1));
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
    // that completes a transaction on the receiver's mbarrier for that row.
    // The warp that reads a pushed row also arms (expect_tx) its barrier.
    const bool push_lo = NB > 1 && yl == 0 && yb > 0;
    const bool push_hi = NB > 1 && yl == BY - 1 && yb < NB - 1;
    uint32_t peer_psi = 0, peer_mbar = 0;
    if (push_lo || push_hi) {
        const uint32_t nb = uint32_t(yb + (push_lo ? -1 : 1));
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(peer_psi) : "r"(smem_u32(psi)), "r"(nb));
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n"
                     : "=r"(peer_mbar)
                     : "r"(smem_u32(&s_mbar[push_lo ? 2 : 0])), "r"(nb));
    }
    constexpr uint32_t ROW_BYTES = uint32_t(E * C * 8);
    auto push_row = [&](int pz, int c, double v) {
        if (!(push_lo || push_hi)) return;
        const int idx = pidx(pz & 3, c, x, push_lo ? BY : -1);
        asm volatile(
            "st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];\n" ::"r"(
                peer_psi + uint32_t(idx) * 8u),
            "l"(__double_as_longlong(v)), "r"(peer_mbar + uint32_t((pz & 1) * 8))
            : "memory");
    };
    // only the rows that read a pushed ring row arm and wait for it (E = 32:
    // one warp per row, so this is warp-uniform)
    const bool needs_rows = NB > 1 && ((yl == 0 && yb > 0) || (yl == BY - 1 && yb < NB - 1));
    const uint32_t my_mbar = smem_u32(&s_mbar[yl == 0 ? 0 : 2]);
    auto expect_rows = [&](int pz) {
        if (needs_rows && (tid & 31) == 0)
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(
                             my_mbar + uint32_t((pz & 1) * 8)),
                         "r"(ROW_BYTES)
                         : "memory");
    };
    auto wait_rows = [&](int pz) {
        if (!needs_rows) return;
        const uint32_t bar = my_mbar + uint32_t((pz & 1) * 8);
        const uint32_t parity = uint32_t((pz >> 1) & 1);
        uint32_t ok = 0;
        while (!ok)
            asm volatile(
                "{\n .reg .pred q;\n mbarrier.try_wait.parity.shared::cta.b64 q, [%1], %2, 1000000;\n"
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
        auto load = [&](int c, double* f) {
            if (sol) {
#pragma unroll
                for (int i = 0; i < Q; ++i) f[i] = 0.0;
            } else if (fast_rows && pz >= 1 && pz <= E - 2) {
                pull_cell_fast<E>(rt_pull, c, x, y, pz, f);
            } else if (mode == MODE_PULL) {
                pull_cell<E>(rt_pull, c, hs, s_solid, x, y, pz, f);
            } else {
                double a0, a1, a2;
                gen_fin<E>(mode, c, s_tc, x, y, pz, f, a0, a1, a2);
            }
            if (!sol) apply_pokes<E>(d, slot, c, x, y, pz, f);
        };
        auto finish = [&](int c, const double* f) {
            double v = 0.0, rho = 0.0;
            if (!sol) {
#pragma unroll
                for (int i = 0; i < Q; ++i) {
                    rho += f[i];
                    negs += f[i] < 0.0;
                }
                if constexpr ((OPT & TM_MEMONLY) != 0) {
                    v = rho;
                } else if (!isfinite(rho)) {
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
            // the P1 density is the P5 density of the same populations (same
            // sum, same order): stashed with them for the collision
            if ((pz & 1) == 0) {
                tm_store20(tbase + uint32_t(c * T::CB), f, rho);
            } else {
                double* st = stage + size_t(c) * (Q + 1) * NT + tid;
#pragma unroll
                for (int i = 0; i < Q; ++i) st[i * NT] = f[i];
                st[Q * NT] = rho;
            }
        };
#pragma unroll 1
        for (int c = 0; c < C; ++c) {
            double f[Q];
            load(c, f);
            finish(c, f);
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
        double Fi[C][3], Fx[C][3];
        bool has_x[C];
        if constexpr ((OPT & TM_MEMONLY) == 0) {
            if (!sol) forces_all<C, PW, PP>(pm, p0, ppl, Fi, Fx, has_x);
        }
#pragma unroll
        for (int c = 0; c < C; ++c) {
            double f[Q], rho;
            if ((z & 1) == 0) {
                tm_load20(tbase + uint32_t(c * T::CB), f, rho);  // warp-convergent
            } else {
                const double* st = stage + size_t(c) * (Q + 1) * NT + tid;
#pragma unroll
                for (int i = 0; i < Q; ++i) f[i] = st[i * NT];
                rho = st[Q * NT];
            }
            if (sol) continue;
            if constexpr ((OPT & TM_MEMONLY) != 0) {
                double* out = fo + c * size_t(Q) * E3 + cell;
                const double ps = p0[c * PP] + pm[c * PP] + ppl[c * PP];
#pragma unroll
                for (int i = 0; i < Q; ++i) out[size_t(i) * E3] = f[i] + ps;
                continue;
            }
            double u0 = 0.0, u1 = 0.0, u2 = 0.0;
            if (mode == MODE_PULL) velocity(f, rho, u0, u1, u2);
            else gen_u<E>(mode, c, s_tc, x, y, z, u0, u1, u2);
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
            // total force in the reference's order: gravity, intra, inter
            const CompConst& kc = P.comp[c];
            double F0 = 0.0, F1 = 0.0, F2 = 0.0;
            if (kc.has_gravity) {
                F0 = rho * kc.gravity[0];
                F1 = rho * kc.gravity[1];
                F2 = rho * kc.gravity[2];
            }
            F0 += Fi[c][0];
            F1 += Fi[c][1];
            F2 += Fi[c][2];
            if (has_x[c]) {
                F0 += Fx[c][0];
                F1 += Fx[c][1];
                F2 += Fx[c][2];
            }
            double* out = fo + c * size_t(Q) * E3 + cell;
            collide_bgk(f, rho, u0, u1, u2, F0, F1, F2, kc.omega, out, size_t(E3), zero_rho);
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
            __syncthreads();
            wait_rows(z + 1);
        } else {
            fill_zghost(E);
            __syncthreads();
        }
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
