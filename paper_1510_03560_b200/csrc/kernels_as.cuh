// kernels_as.cuh — k_main_as: the asynchronously staged fused step kernel.
//
// What bounds the TMEM-stash kernel (k_main_tm) is not the arithmetic and not
// the access pattern — a copy kernel with the same 38 shifted SoA streams per
// column block runs at the flat-copy rate (tools/bwtest.cu) — but memory-level
// parallelism: its pulls are synchronous register loads, so every plane costs
// two or three DRAM round trips that only 16 warps per SM can overlap.
//
// k_main_as decouples the pulls from the arithmetic:
//   * every population of plane pz is requested with cp.async (8 B per cell
//     and direction, the same pull rules) into a shared-memory landing
//     buffer two planes before the psi pass reads it, together with the psi
//     ghost entries of that plane (x ring, tile-edge halo rows) straight into
//     the psi ring;
//   * the psi pass reads the landed populations, computes rho -> psi and
//     moves them (with rho) into Tensor Memory, where they wait for the
//     collision one plane later (two TMEM plane slots, 160 columns at C = 2);
//   * CTA = 32 x 4 column block (4 warps, one row each), cluster = the 8
//     blocks of a 32^3 tile exchanging psi edge rows through DSMEM (st.async +
//     mbarrier, as k_main_tm); two CTAs per SM at up to 255 registers, so the
//     two components' dependency chains interleave without spills.
// Per plane z:  wait landing(z+1) | psi pass z+1 -> TMEM | issue(z+3)
//               | CTA barrier | edge rows wait | collide z from TMEM.
#pragma once

#include "kernels_tm.cuh"

namespace plbm {

template <int E, int C>
struct AsCfg {
    static constexpr int NT = 128;
    static constexpr int BY = NT / E;     // rows per CTA
    static constexpr int NB = E / BY;     // CTAs per tile = cluster size
    static constexpr int CB = 40;         // TMEM columns per (plane slot, component)
    static constexpr int NCOLS = (2 * C * CB <= 128) ? 128 : 256;
    static constexpr int PW = E + 2;
    static constexpr int PH = BY + 2;
    static constexpr int PP = PW * PH;
    static constexpr int RING = 8;        // psi planes z-2 .. z+3 live (+2 spare)
    static constexpr int PSI_BYTES = RING * C * PP * 8;
    static constexpr int LAND_BYTES = 2 * C * Q * NT * 8;  // two landing planes
    static constexpr int SMEM = PSI_BYTES + LAND_BYTES;
    static_assert(2 * C * CB <= NCOLS, "TMEM plane slots do not fit");
    static_assert(2 * (SMEM + 8 * 1024) <= 228 * 1024, "two CTAs per SM must fit");
};

__device__ __forceinline__ void cp_async8(uint32_t dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// psi_ghost (kernels.cuh) split into "load this address" or "use this value".
template <int E>
__device__ __forceinline__ const double* psi_ghost_src(const RouteTab& rt, int c, bool hs,
                                                       const uint32_t* sb, int x, int y, int z,
                                                       double& val) {
    if (hs && solid_at<E>(sb, x, y, z)) {
        val = 0.0;
        return nullptr;
    }
    const int ox = x < 0 ? -1 : (x >= E ? 1 : 0);
    const int oy = y < 0 ? -1 : (y >= E ? 1 : 0);
    const int oz = z < 0 ? -1 : (z >= E ? 1 : 0);
    const int pat = (ox + 1) + 3 * (oy + 1) + 9 * (oz + 1);
    if (rt.nb[pat]) {
        val = P.comp[c].psi_nb;
        return nullptr;
    }
    int face;
    if (ox) face = ox > 0 ? 0 : 1;
    else if (oy) face = oy > 0 ? 2 : 3;
    else face = oz > 0 ? 4 : 5;
    const int lx = x & (E - 1), ly = y & (E - 1), lz = z & (E - 1);
    constexpr int E2 = E * E;
    return rt.p[pat] + (size_t(c) * 6 + face) * E2 + face_index<E>(face, lx, ly, lz);
}

template <int E, int C>
__global__ void __launch_bounds__(128, 2) k_main_as(Dev d, const int* __restrict__ active,
                                                    int src_buf, int write_uface, long iter) {
    using T = AsCfg<E, C>;
    constexpr int NT = T::NT, BY = T::BY, NB = T::NB, PW = T::PW, PH = T::PH, PP = T::PP;
    constexpr int R = T::RING;
    constexpr int G = E + 2;
    constexpr int E2 = E * E;
    constexpr int E3 = E * E * E;
    static_assert(NB == 1 || (BY * E == NT && (E == 32 || BY % 2 == 0)), "block rows");
    extern __shared__ __align__(16) double smem[];
    double* psi = smem;                 // [R][C][PH][PW] ring of psi planes
    double* land = smem + R * C * PP;   // [2][C][Q][NT] landed populations
    __shared__ RouteTab rt_pull, rt_psi;
    __shared__ uint32_t s_solid[(G * G * G + 31) / 32];
    __shared__ int s_tc[3];
    __shared__ uint32_t s_tmem;
    __shared__ __align__(8) uint64_t s_mbar[4];  // pushed rows: [0..1] row -1, [2..3] row BY

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
        for (int k = 0; k < 4; ++k)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(&s_mbar[k])), "r"(1));
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    if constexpr (NB > 1) {  // peers see our initialised mbarriers before pushing rows
        asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
        asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
    }
    // 4 warps: warp w owns TMEM lanes 32w..32w+31
    const uint32_t tbase = s_tmem + (uint32_t(32 * warp) << 16);
    const int tile_lin = (s_tc[0] * P.grid[1] + s_tc[1]) * P.grid[2] + s_tc[2];

    const int x = tid % E;
    const int yl = tid / E;
    const int y = y0 + yl;
    // E = 32: one warp per row, so every per-row test below is warp-uniform
    const bool fast_rows = mode == MODE_PULL && !hs && y >= 1 && y <= E - 2;
    auto pidx = [&](int pz, int c, int xx, int yy_local) {
        return (((pz & (R - 1)) * C + c) * PH + (yy_local + 1)) * PW + (xx + 1);
    };
    const uint32_t land_u32 = smem_u32(land);
    auto land_addr = [&](int pz, int c, int i) {  // this thread's landing slot
        return land_u32 + uint32_t((((pz & 1) * C + c) * Q + i) * NT + tid) * 8u;
    };

    // ---- cluster psi-row exchange (see k_main_tm) ----------------------------
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
        const int idx = pidx(pz, c, x, push_lo ? BY : -1);
        asm volatile(
            "st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];\n" ::"r"(
                peer_psi + uint32_t(idx) * 8u),
            "l"(__double_as_longlong(v)), "r"(peer_mbar + uint32_t((pz & 1) * 8))
            : "memory");
    };
    const bool needs_rows = NB > 1 && ((yl == 0 && yb > 0) || (yl == BY - 1 && yb < NB - 1));
    const uint32_t my_mbar = smem_u32(&s_mbar[yl == 0 ? 0 : 2]);
    auto expect_rows = [&](int pz) {
        if (needs_rows && x == 0)  // one lane of the reading row arms its barrier
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
                "{\n .reg .pred q;\n mbarrier.try_wait.parity.shared::cta.b64 q, [%1], %2;\n"
                " selp.u32 %0, 1, 0, q;\n}\n"
                : "=r"(ok)
                : "r"(bar), "r"(parity)
                : "memory");
    };

    // ---- psi ghost entries ------------------------------------------------------
    auto fill_zghost = [&](int pz) {  // whole plane outside the tile in z (synchronous)
        for (int k = tid; k < PP; k += NT) {
            const int xx = k % PW - 1, yy = k / PW - 1 + y0;
            const bool xo = xx < 0 || xx >= E, yo = yy < 0 || yy >= E;
#pragma unroll 1
            for (int c = 0; c < C; ++c)
                psi[pidx(pz, c, xx, yy - y0)] =
                    (xo && yo) ? 0.0 : psi_ghost<E>(rt_psi, c, hs, s_solid, xx, yy, pz);
        }
    };
    // x ring + tile-edge halo rows of plane pz, landed asynchronously
    auto issue_ring = [&](int pz) {
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
            for (int c = 0; c < C; ++c) {
                double v;
                const double* src = psi_ghost_src<E>(rt_psi, c, hs, s_solid, xx, y0 + yyl, pz, v);
                const int idx = pidx(pz, c, xx, yyl);
                if (src) cp_async8(smem_u32(psi + idx), src);
                else psi[idx] = v;
            }
        }
    };

    // ---- issue(pz): every population the psi pass of plane pz pulls ---------
    auto issue = [&](int pz) {
        if (pz < E) {
            if (mode == MODE_PULL && !(hs && solid_at<E>(s_solid, x, y, pz))) {
#pragma unroll 1
                for (int c = 0; c < C; ++c) {
                    if (fast_rows && pz >= 1 && pz <= E - 2)
                        pull_addr_fast<E>(rt_pull, c, x, y, pz,
                                          [&](int i, const double* p) { cp_async8(land_addr(pz, c, i), p); });
                    else
                        pull_addr<E>(rt_pull, c, hs, s_solid, x, y, pz,
                                     [&](int i, const double* p) { cp_async8(land_addr(pz, c, i), p); });
                }
            }
            issue_ring(pz);
        }
        cp_async_commit();  // one group per plane (empty past the last plane)
    };

    // ---- psi pass of plane pz: landed f -> rho -> psi, stash in TMEM ---------
    auto psi_pass = [&](int pz) {
        const bool sol = hs && solid_at<E>(s_solid, x, y, pz);
        int negs = 0, clamps = 0;
        double f[C][Q], rho[C];
#pragma unroll
        for (int c = 0; c < C; ++c) {
            if (sol) {
#pragma unroll
                for (int i = 0; i < Q; ++i) f[c][i] = 0.0;
            } else if (mode == MODE_PULL) {
                const double* l = land + size_t(((pz & 1) * C + c) * Q) * NT + tid;
#pragma unroll
                for (int i = 0; i < Q; ++i) f[c][i] = l[i * NT];
            } else {
                double a0, a1, a2;
                gen_fin<E>(mode, c, s_tc, x, y, pz, f[c], a0, a1, a2);
            }
            rho[c] = 0.0;
        }
#pragma unroll
        for (int c = 0; c < C; ++c) {
            double v = 0.0;
            if (!sol) {
#pragma unroll
                for (int i = 0; i < Q; ++i) {
                    rho[c] += f[c][i];
                    negs += f[c][i] < 0.0;
                }
                if (!isfinite(rho[c])) {
                    atomic_err(d.err, iter, tile_lin, ERR_P1_NAN);
                } else {
                    double press;
                    if (!pr_pressure(rho[c], P.comp[c], press)) {
                        atomic_err(d.err, iter, tile_lin, ERR_P1_POLE);
                    } else {
                        bool cl;
                        v = pseudo_potential(rho[c], press, P.comp[c], cl);
                        clamps += cl;
                    }
                }
            }
            psi[pidx(pz, c, x, yl)] = v;
            push_row(pz, c, v);
            // the P1 density is the P5 density of the same populations
            tm_store20(tbase + uint32_t(((pz & 1) * C + c) * T::CB), f[c], rho[c]);
        }
        asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
        const unsigned m1 = __reduce_add_sync(0xffffffffu, (unsigned)negs);
        const unsigned m2 = __reduce_add_sync(0xffffffffu, (unsigned)clamps);
        if ((tid & 31) == 0) {
            if (m1) atomicAdd(&d.cnt[CNT_NEG], (unsigned long long)m1);
            if (m2) atomicAdd(&d.cnt[CNT_CLAMP], (unsigned long long)m2);
        }
    };

    // ---- collide plane z from TMEM -------------------------------------------
    auto collide_plane = [&](int z) {
        const bool sol = hs && solid_at<E>(s_solid, x, y, z);
        const int cell = (z * E + y) * E + x;
        const double* pm = psi + pidx(z - 1, 0, x, yl);
        const double* p0 = psi + pidx(z, 0, x, yl);
        const double* ppl = psi + pidx(z + 1, 0, x, yl);
        constexpr int CP = PP;  // component stride inside one ring plane
        unsigned fmask = 0;
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
        if (!sol) forces_all<C, PW, CP>(pm, p0, ppl, Fi, Fx, has_x);
#pragma unroll
        for (int c = 0; c < C; ++c) {
            double f[Q], rho;
            tm_load20(tbase + uint32_t(((z & 1) * C + c) * T::CB), f, rho);  // warp-convergent
            if (sol) continue;
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
                cp[cell] = p0[c * CP];
                cp[E3 + cell] = u0;
                cp[2 * E3 + cell] = u1;
                cp[3 * E3 + cell] = u2;
            }
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

    // ---- pipeline -------------------------------------------------------------
    issue(0);
    issue(1);
    fill_zghost(-1);
    expect_rows(0);
    cp_async_wait<1>();  // plane 0 landed (this thread's slots)
    __syncthreads();     // ... and every thread's ring entries of plane 0
    psi_pass(0);
    issue(2);
    __syncthreads();
    wait_rows(0);
#pragma unroll 1
    for (int z = 0; z < E; ++z) {
        if (z + 1 < E) {
            expect_rows(z + 1);
            cp_async_wait<1>();  // plane z+1 landed; plane z+2 may still be in flight
            psi_pass(z + 1);
            issue(z + 3);        // reuses plane z+1's landing slots (read above)
        } else {
            fill_zghost(E);
        }
        __syncthreads();  // psi plane z+1 (and its ghost ring) visible CTA-wide
        if (z + 1 < E) wait_rows(z + 1);
        collide_plane(z);
    }
    cp_async_wait<0>();
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
