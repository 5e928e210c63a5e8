// kernels_pc.cuh — k_main_pc: one CTA per (column block, component), with the
// pulls staged asynchronously.
//
// Measured constraints that shape it (profiles/, tools/bwtest.cu):
//   * the 38 shifted SoA streams of a column block stream at the flat-copy
//     rate when enough bytes are in flight — the access pattern is not the
//     limit, memory-level parallelism is;
//   * the FP64 work needs ~16 warps per SM to hide its dependency chains (a
//     cp.async-staged two-components-per-thread variant at 8 warps/SM was
//     latency-bound on arithmetic: 4.9 ms vs 3.6 ms for k_main_tm);
//   * at 16 warps/SM and two components per thread there is no room on chip
//     for a landing buffer next to the two-plane stash.
// Splitting the components over the two CTAs of a cluster pair halves the
// per-CTA population state, which buys both: at 16 warps per SM each thread
// holds one cell of one component, its next plane lands in shared memory by
// cp.async while the current plane collides, and the stash of two planes
// lives in Tensor Memory (2 x 40 columns).  psi values cross to the partner
// component's CTA (whole plane) and to the y-neighbour blocks (edge rows, both
// components) through distributed shared memory with st.async, completing
// transactions on the receiver's per-plane mbarrier.
//
// Cluster = NB / NH y-blocks x C components of one tile: NH = 1 is the whole
// tile (E = 32: 4 x 2 = 8 CTAs; 12 at C = 3, a non-portable size B200
// supports), NH = 2 / 4 split it (the default NH = 4: 2-CTA clusters at
// E = 32, C = 2, which fill every SM slot; psi across the split boundaries
// from the face pass's mid faces, see k_main_pc).
// Per plane z:  wait landing(z+1) | psi pass z+1 -> TMEM, push psi | issue
//               pulls(z+2) | CTA barrier | issue ghosts(z+2) | wait pushes(z+1)
//               | collide z from TMEM.
#pragma once

#include "physics.cuh"

namespace plbm {

static __constant__ unsigned char c_xdir[XN] = {0, 2, 3, 4, 5, 6, 8, 10, 12, 14, 15, 16, 17, 18, 2, 8, 10, 12, 14,
                                         1, 7, 9, 11, 13, 0, 1, 3, 4, 5, 6, 7, 9, 11, 13, 15, 16, 17, 18};

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


template <int E, int C, int LAG = 1, int NT_ = 256, int NH_ = 1>
struct PcCfg {
    static constexpr int NT = NT_;      // 256: 8 warps, 2 CTAs/SM; 512 (E = 64): 16 warps, 1 CTA/SM
    static constexpr int BY = NT / E;   // rows per CTA
    static constexpr int NB = E / BY;   // y-blocks per tile
    static constexpr int NH = NH_;      // clusters per tile (tile halves along y)
    static constexpr int NBC = NB / NH; // y-blocks per cluster
    static constexpr int CL = NBC * C;  // cluster size
    static_assert(NB % NH == 0, "clusters split a tile's y-blocks evenly");
    static constexpr int CB = 40;       // TMEM columns per plane slot (19 f + rho)
    static constexpr int WPQ = NT / 128;  // warps per TMEM lane quarter
    static constexpr int NCOLS = 128 * WPQ;  // 128 columns per thread
    static constexpr int PW = E + 2;
    static constexpr int PH = BY + 2;
    static constexpr int PP = PW * PH;
    static constexpr int RING = LAG == 1 ? 4 : 8;  // psi planes z-2 .. z+LAG+1 live
    static constexpr int NMB = 2 * LAG;             // pushed-plane mbarriers
    static constexpr int TSLOTS = LAG + 1;          // TMEM plane slots
    static constexpr int PSI_BYTES = RING * C * PP * 8;
    static constexpr int LAND_BYTES = Q * NT * 8;
    static constexpr int XST_BYTES = 2 * 4 * Q * BY * 8;  // x-column staging, two planes
    static constexpr int SMEM = PSI_BYTES + LAND_BYTES + XST_BYTES;
    static_assert(CL <= 16, "cluster size (> 8 needs the non-portable opt-in)");
    static_assert(TSLOTS * CB <= NCOLS / WPQ, "TMEM plane slots do not fit");
    static constexpr int PER_SM = 512 / NT;  // 16 warps per SM
    // static shared memory: the extended-grid solid mask + route tables etc.
    static constexpr int STATIC_EST = ((E + 2) * (E + 2) * (E + 2) + 31) / 32 * 4 + 3 * 1024;
    static_assert(PER_SM * (SMEM + STATIC_EST + 1024) <= 228 * 1024, "CTAs per SM must fit");
};

// LAG = planes between a plane's psi pass and its collision: 1 (psi of z+1
// is computed and pushed in the iteration that collides z) or 2 (pushed one
// iteration before it is needed, three TMEM plane slots).
// EARLY: the thread-local head of the collision of plane z (TMEM load of f
// and rho, u = m / rho) runs before the wait for the peers' psi of plane z+1,
// overlapping the divisions with the cluster synchronisation.
// MEMONLY (probe, variant 24, NOT a correct step): the same pulls, psi
// pushes, TMEM stash, stores and xcol staging with the physics removed (psi
// = 0, f stored unchanged) — the memory pipeline's own ceiling.
// AA: population storage kind of this step (kernels.cuh AA_*).
// NH > 1: a cluster covers 1/NH of the tile's y-blocks (fewer CTAs per
// cluster: 2 instead of 8 at E = 32, C = 2, NH = 4, which pack the SMs
// better); the psi rows across a cluster boundary come from the mid-face
// buffers the previous step's face pass wrote (face_xyz faces 6..), as
// tile-edge rows come from the neighbours' face buffers.
template <int E, int C, int LAG, int NT_ = 256, bool EARLY = true, bool MEMONLY = false, int AA = AA_OFF,
          int NH = 1>
__global__ void __launch_bounds__(NT_, 512 / NT_) k_main_pc(Dev d, const int* __restrict__ active,
                                                            int src_buf, int write_uface, long iter) {
    if (halted(d)) return;
    const unsigned long long t_start = d.probe ? global_ns() : 0ull;
    using T = PcCfg<E, C, LAG, NT_, NH>;
    constexpr int NMB = T::NMB;
    constexpr int NT = T::NT, BY = T::BY, NBC = T::NBC, PW = T::PW, PH = T::PH, PP = T::PP;
    constexpr int R = T::RING;
    constexpr int G = E + 2;
    constexpr int E2 = E * E;
    constexpr int E3 = E * E * E;
    extern __shared__ __align__(16) double smem[];
    double* psi = smem;                // [R][C][PH][PW] ring of psi planes, all components
    double* land = smem + R * C * PP;  // [Q][NT] landed populations of the next plane
    double* xst = land + Q * NT;       // [2][4][Q][BY] x-column values of the block's rows, by plane parity
    __shared__ RouteTab rt_pull, rt_psi, rt_w;
    __shared__ uint32_t s_solid[(G * G * G + 31) / 32];
    __shared__ int s_tc[3];
    __shared__ uint32_t s_tmem;
    __shared__ __align__(8) uint64_t s_mbar[T::NMB];  // pushed psi of plane p: slot p % NMB
    __shared__ int s_ready[20], s_nready;              // fused face pass: tiles this cluster runs

    const int tid = threadIdx.x;
    const int warp = tid >> 5;
    const int rank = int(blockIdx.x % T::CL);  // = cluster CTA rank (1-D clusters)
    const int tile_i = int(blockIdx.x / T::CL) / NH;
    // (interleaving the components in the rank order measured no different:
    // the 8 CTAs of a cluster sit on 8 different SMs, tools/probe_cluster.py)
    const int c = rank / NBC;                  // this CTA's component
    const int ybl = rank % NBC;                // y-block within the cluster
    const int yb = int(blockIdx.x / T::CL) % NH * NBC + ybl;
    auto crank = [&](int cc, int bb) { return cc * NBC + bb; };
    const int y0 = yb * BY;
    if (d.nactive && d.tile_base + tile_i >= *d.nactive) return;  // (whole clusters: same tile)
    const int slot = active[tile_i];
    if (d.no_fluid && d.no_fluid[slot] && !(d.face_flags & FACE_FUSED)) return;  // (whole clusters: same tile)
    const uint8_t mode = d.mode[slot];
    const bool hs = d.has_solid[slot] != 0;
    const int amb = P.amb_slot;
    const int par = int(iter & 1);
    double* __restrict__ fo = d.slot_f[src_buf ^ 1][slot] + size_t(c) * Q * E3;
    const int li = d.lidx[slot];

    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                         smem_u32(&s_tmem)),
                     "n"(T::NCOLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    load_routes(rt_pull, d.route[ROUTE_PULL] + size_t(slot) * 18, slot, amb, d.slot_f[src_buf]);
    load_routes(rt_psi, d.route[ROUTE_PSI] + size_t(slot) * 18, slot, amb, d.slot_pf[par], d.mode);
    if constexpr (AA == AA_NEIGH) load_routes(rt_w, d.route[ROUTE_W] + size_t(slot) * 18, slot, amb, d.slot_f[0]);
    if (tid < 3) s_tc[tid] = d.coords[slot * 3 + tid];
    if (hs)
        for (int k = tid; k < d.solid_words; k += NT) s_solid[k] = d.solid[size_t(slot) * d.solid_words + k];
    if (tid == 0) {
        for (int k = 0; k < NMB; ++k)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(&s_mbar[k])), "r"(1));
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    if constexpr (T::CL > 1) {  // peers see our initialised mbarriers before pushing
        asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
        asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
    }
    // 8 warps: warps w and w+4 share TMEM lanes 32(w%4).., split by columns
    const uint32_t tbase = s_tmem + (uint32_t(32 * (warp & 3)) << 16) + uint32_t((warp >> 2) * 128);
    const int tile_lin = (s_tc[0] * P.grid[1] + s_tc[1]) * P.grid[2] + s_tc[2];

    const int x = tid % E;
    const int yl = tid / E;
    const int y = y0 + yl;
    const int xcls = x == 0 ? 0 : x == 1 ? 1 : x == E - 2 ? 2 : x == E - 1 ? 3 : -1;  // xcol lanes
    double* const xcol = d.slot_f[src_buf ^ 1][slot] + size_t(C) * Q * E3 + size_t(c) * XN * E2;
    // xcol holds f_post of the boundary columns — the A-B pull's values — so
    // the face pass reads it the same way whatever the storage kind
    const bool wx = d.xcol_ok != 0;
    // xcol: the x-column lanes stage their values in shared memory during the
    // collision; after the next CTA barrier the block writes them out as
    // 8-row (64-byte) segments of xcol[c][slot][z][y]
    auto flush_xcol = [&](int pz) {
        if (!wx || pz < 0) return;
        const double* src = xst + (pz & 1) * 4 * Q * BY;
        // items beyond NT land on warps 2-3 (warp 0 polls the mbarrier, warps
        // 0 / BY-1 are the tile-edge rows of the edge blocks)
        for (int k = (tid + NT - 64) % NT; k < XN * BY; k += NT) {
            const int s = k / BY, r = k - s * BY;
            xcol[size_t(s) * E2 + pz * E + y0 + r] = src[(xslot_cls(s) * Q + c_xdir[s]) * BY + r];
        }
    };
    const bool fast_rows = mode == MODE_PULL && !hs && y >= 1 && y <= E - 2;
    const bool fast_yedge = mode == MODE_PULL && !hs && !fast_rows;  // y == 0 or E-1
    auto pidx = [&](int pz, int cc, int xx, int yy_local) {
        return (((pz & (R - 1)) * C + cc) * PH + (yy_local + 1)) * PW + (xx + 1);
    };
    const uint32_t land_u32 = smem_u32(land);
    // frontier faces this cell's column lies on (criterion u_prev, u_face):
    // x/y faces are fixed per thread, z faces apply to the first/last plane
    unsigned xy_fmask = 0, z_fmask = 0;
    if (write_uface) {
        if (x == 0 && rt_psi.s[face_pattern(0)] == amb) xy_fmask |= 1u;
        if (x == E - 1 && rt_psi.s[face_pattern(1)] == amb) xy_fmask |= 2u;
        if (y == 0 && rt_psi.s[face_pattern(2)] == amb) xy_fmask |= 4u;
        if (y == E - 1 && rt_psi.s[face_pattern(3)] == amb) xy_fmask |= 8u;
        if (rt_psi.s[face_pattern(4)] == amb) z_fmask |= 16u;
        if (rt_psi.s[face_pattern(5)] == amb) z_fmask |= 32u;
    }

    // ---- psi pushes: whole plane to the other components' CTAs of this block,
    // edge rows to every component's CTA of the adjacent y-blocks ------------
    const uint32_t psi_u32 = smem_u32(psi);
    const uint32_t mbar_u32 = smem_u32(&s_mbar[0]);
    auto push = [&](int dst_rank, int pz, int yy_local, double v) {
        uint32_t ra, rb;
        asm("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(ra) : "r"(psi_u32), "r"(dst_rank));
        asm("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(rb) : "r"(mbar_u32), "r"(dst_rank));
        asm volatile(
            "st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];\n" ::"r"(
                ra + uint32_t(pidx(pz, c, x, yy_local)) * 8u),
            "l"(__double_as_longlong(v)), "r"(rb + uint32_t((pz & (NMB - 1)) * 8))
            : "memory");
    };
    auto push_all = [&](int pz, double v) {
#pragma unroll
        for (int c2 = 0; c2 < C; ++c2) {
            if (c2 != c) push(crank(c2, ybl), pz, yl, v);
            if (yl == 0 && ybl > 0) push(crank(c2, ybl - 1), pz, BY, v);
            if (yl == BY - 1 && ybl < NBC - 1) push(crank(c2, ybl + 1), pz, -1, v);
        }
    };
    constexpr uint32_t PLANE_BYTES = uint32_t((C - 1) * BY * E * 8);
    const uint32_t expect_bytes =
        PLANE_BYTES + uint32_t(((ybl > 0) + (ybl < NBC - 1)) * C * E * 8);
    auto expect = [&](int pz) {
        if (T::CL > 1 && tid == 0)
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(
                             mbar_u32 + uint32_t((pz & (NMB - 1)) * 8)),
                         "r"(expect_bytes)
                         : "memory");
    };
    // the warp that polls the mbarrier: a middle row (no tile-edge pushes), no
    // ring issue (warps RT0/32 ..), no xcol-flush remainder (warps 2-3)
    constexpr int POLL_WARP = NT / 32 - 3;
    auto wait_pushed = [&](int pz) {
        if (T::CL == 1) return;
        const uint32_t bar = mbar_u32 + uint32_t((pz & (NMB - 1)) * 8);
        const uint32_t parity = uint32_t((pz / NMB) & 1);
        uint32_t ok = 0;
        while (!ok)
            asm volatile(
                "{\n .reg .pred q;\n mbarrier.try_wait.parity.shared::cta.b64 q, [%1], %2, 1000000;\n"
                " selp.u32 %0, 1, 0, q;\n}\n"
                : "=r"(ok)
                : "r"(bar), "r"(parity)
                : "memory");
    };

    // ---- psi ghost entries (both components) ---------------------------------
    auto fill_zghost = [&](int pz) {
        for (int k = tid; k < PP; k += NT) {
            const int xx = k % PW - 1, yy = k / PW - 1 + y0;
            const bool xo = xx < 0 || xx >= E, yo = yy < 0 || yy >= E;
#pragma unroll 1
            for (int cc = 0; cc < C; ++cc)
                psi[pidx(pz, cc, xx, yy - y0)] =
                    (xo && yo) ? 0.0 : psi_ghost<E>(rt_psi, cc, hs, s_solid, xx, yy, pz);
        }
    };
    auto issue_ring = [&](int pz) {  // x ring + tile-edge halo rows, asynchronously
        if (pz >= E) return;
        // run by the middle warps (never the poller, never a tile-edge row)
        constexpr int RITEMS = 2 * PH + 2 * E;
        constexpr int RT0 = NT > RITEMS ? ((NT - RITEMS) / 2) & ~31 : 0;
        for (int k = tid - RT0; k < RITEMS; k += NT) {
            if (k < 0) continue;
            int xx, yyl;
            if (k < 2 * PH) {
                xx = (k & 1) ? E : -1;
                yyl = (k >> 1) - 1;
            } else {
                const int q = k - 2 * PH;
                xx = q % E;
                yyl = (q / E) ? BY : -1;
                const int yy = y0 + yyl;
                if (yy >= 0 && yy < E) {
                    if (yyl < 0 ? ybl > 0 : ybl < NBC - 1) continue;  // pushed by the adjacent y-block
                    // across a cluster boundary: the mid-face buffers (face_xyz faces 6..)
                    const int m = 2 * ((yyl < 0 ? y0 : yy) / P.mid_sp - 1) + (yyl < 0 ? 0 : 1);
#pragma unroll 1
                    for (int cc = 0; cc < C; ++cc) {
                        const int idx = pidx(pz, cc, xx, yyl);
                        if (hs && solid_at<E>(s_solid, xx, yy, pz)) psi[idx] = 0.0;
                        else if (rt_psi.nb[13]) psi[idx] = P.comp[cc].psi_nb;  // newborn: ambient cells
                        else
                            cp_async8(smem_u32(psi + idx), rt_psi.p[13] +
                                                               (size_t(C) * 6 + cc * d.mid_faces + m) * E2 +
                                                               xx + E * pz);
                    }
                    continue;
                }
            }
#pragma unroll 1
            for (int cc = 0; cc < C; ++cc) {
                double v;
                const double* src = psi_ghost_src<E>(rt_psi, cc, hs, s_solid, xx, y0 + yyl, pz, v);
                const int idx = pidx(pz, cc, xx, yyl);
                if (src) cp_async8(smem_u32(psi + idx), src);
                else psi[idx] = v;
            }
        }
    };
    auto issue_pulls = [&](int pz) {
        if (pz >= E || mode != MODE_PULL || (hs && solid_at<E>(s_solid, x, y, pz))) return;
        auto op = [&](int i, const double* p) { cp_async8(land_u32 + uint32_t(i * NT + tid) * 8u, p); };
        if constexpr (AA != AA_OFF) {
            if (mode == MODE_PULL && !hs && pz >= 1 && pz <= E - 2) pull_addr_row_aa<E, AA>(rt_pull, c, x, y, pz, op);
            else pull_addr<E, AA>(rt_pull, c, hs, s_solid, x, y, pz, op);
        } else if (fast_rows && pz >= 1 && pz <= E - 2) pull_addr_fast<E>(rt_pull, c, x, y, pz, op);
        else if (fast_yedge && pz >= 1 && pz <= E - 2) pull_addr_fast_yedge<E>(rt_pull, c, x, y, pz, op);
        else pull_addr<E>(rt_pull, c, hs, s_solid, x, y, pz, op);
    };

    // Per-thread diagnostics, reduced once at the end of the kernel.
    // Negative populations: when every population this step can pull passed
    // the previous step's screen (no tile marked; the constants checked on
    // the host; no poke), none is -0, NaN or subnormal, so f < 0 is exactly
    // its sign bit — an integer op instead of an FP64 compare per value.
    unsigned negs = 0, clamps = 0, zero_rho = 0;
    int suspect = 0;
    const bool neg_exact = d.neg_exact || d.npoke || !d.susp_any || d.susp_any[(iter - 1) & 1] != 0u;

    // ---- psi pass of plane pz ---------------------------------------------------
    auto psi_pass = [&](int pz) {
        const bool sol = hs && solid_at<E>(s_solid, x, y, pz);
        double f[Q];
        double v = 0.0, rho = 0.0;
        if (sol) {
#pragma unroll
            for (int i = 0; i < Q; ++i) f[i] = 0.0;
        } else {
            if (mode == MODE_PULL) {
#pragma unroll
                for (int i = 0; i < Q; ++i) f[i] = land[i * NT + tid];
            } else {
                double a0, a1, a2;
                gen_fin<E>(mode, c, s_tc, x, y, pz, f, a0, a1, a2);
            }
            apply_pokes<E>(d, slot, c, x, y, pz, f);
#pragma unroll
            for (int i = 0; i < Q; ++i) rho += f[i];
            if (neg_exact) {
#pragma unroll
                for (int i = 0; i < Q; ++i) negs += f[i] < 0.0;
            } else {
#pragma unroll
                for (int i = 0; i < Q; ++i) negs += uint32_t(__double2hiint(f[i])) >> 31;
            }
            if (MEMONLY) {
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
        psi[pidx(pz, c, x, yl)] = v;
        push_all(pz, v);
        tm_store20(tbase + uint32_t((pz % T::TSLOTS) * T::CB), f, rho);
        asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
    };

    // ---- collide plane z (this CTA's component) ------------------------------
    // head: f and rho from TMEM, u (thread-local; no psi needed)
    auto collide_head = [&](int z, double (&f)[Q], double& rho, double& u0, double& u1, double& u2) {
        const bool sol = hs && solid_at<E>(s_solid, x, y, z);
        tm_load20(tbase + uint32_t((z % T::TSLOTS) * T::CB), f, rho);  // warp-convergent
        u0 = u1 = u2 = 0.0;
        if (!sol && !MEMONLY) {
            if (mode == MODE_PULL) velocity(f, rho, u0, u1, u2);
            else gen_u<E>(mode, c, s_tc, x, y, z, u0, u1, u2);
        }
    };
    auto collide_plane = [&](int z, double (&f)[Q], double rho, double u0, double u1, double u2) {
        const bool sol = hs && solid_at<E>(s_solid, x, y, z);
        const int cell = (z * E + y) * E + x;
        const double* pm = psi + pidx(z - 1, 0, x, yl);
        const double* p0 = psi + pidx(z, 0, x, yl);
        const double* ppl = psi + pidx(z + 1, 0, x, yl);
        constexpr int CP = PP;
        if (MEMONLY) {
            double* xc = (xcls >= 0 && wx) ? xst + ((z & 1) * 4 + xcls) * Q * BY + yl : nullptr;
#pragma unroll
            for (int i = 0; i < Q; ++i) {
                fo[cell + size_t(i) * E3] = f[i];
                if (xc) xc[i * BY] = f[i];
            }
        } else if (!sol) {
            // forces (engine.cpp:420-449): intra of c, inter from the other
            // component's s1 (the same sum as its intra s1)
            double s1[3], s2[3];
            sc_sums<PW, true>(pm + c * CP, p0 + c * CP, ppl + c * CP, s1, s2);
            const CompConst& kc = P.comp[c];
            const double c1 = kc.c1f * p0[c * CP];
            double F0 = 0.0, F1 = 0.0, F2 = 0.0;
            if (kc.has_gravity) {
                F0 = rho * kc.gravity[0];
                F1 = rho * kc.gravity[1];
                F2 = rho * kc.gravity[2];
            }
            F0 += c1 * s1[0] + kc.c2 * s2[0];
            F1 += c1 * s1[1] + kc.c2 * s2[1];
            F2 += c1 * s1[2] + kc.c2 * s2[2];
#pragma unroll
            for (int c2 = 0; c2 < C; ++c2) {  // inter_force in c2 order (C <= 2: one term)
                if (c2 == c) continue;
                const double g = P.coupling[c * C + c2];
                if (g == 0.0) continue;
                double t[3];
                sc_sums<PW, false>(pm + c2 * CP, p0 + c2 * CP, ppl + c2 * CP, t, nullptr);
                const double cc = (-g) * p0[c * CP];
                F0 += cc * t[0];
                F1 += cc * t[1];
                F2 += cc * t[2];
            }
            const unsigned fmask = xy_fmask | (z == 0 ? z_fmask & 16u : 0u) | (z == E - 1 ? z_fmask & 32u : 0u);
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
            StoreF<E, AA> st{fo + cell, &rt_w, c, x, y, z, hs, s_solid};
            if constexpr (AA == AA_NEIGH) {
                if (mode == MODE_PULL && !hs && z >= 1 && z <= E - 2) {
                    constexpr size_t cs = size_t(Q) * E3;
                    const int row = (z * E + y) * E;
                    auto nb = [&](int pat, int off) -> double* {
                        return rt_w.s[pat] == amb ? nullptr : const_cast<double*>(rt_w.p[pat]) + c * cs + row + off;
                    };
                    const int oy = y == E - 1 ? 1 : -1;   // the row across the y edge (edge rows)
                    const int wrap = y == E - 1 ? -E2 : E2;
                    st.fast = true;
                    st.xm = x == 0 ? nb(12, E - 1) : nullptr;
                    st.xp = x == E - 1 ? nb(14, 0) : nullptr;
                    st.yo = (y == 0 || y == E - 1) ? nb(13 + 3 * oy, x + wrap) : nullptr;
                    st.yxm = x == 0 ? nb(12 + 3 * oy, E - 1 + wrap) : (st.yo ? st.yo - 1 : nullptr);
                    st.yxp = x == E - 1 ? nb(14 + 3 * oy, wrap) : (st.yo ? st.yo + 1 : nullptr);
                }
            }
            collide_bgk(f, rho, u0, u1, u2, F0, F1, F2, kc.omega, st, zero_rho, suspect,
                        (xcls >= 0 && wx) ? xst + ((z & 1) * 4 + xcls) * Q * BY + yl : nullptr, BY);
        }
    };

    // ---- pipeline -------------------------------------------------------------
#ifdef PLBM_PHASES  // measurement build: per-warp cycle accounting of the plane loop
    unsigned long long ph_acc[8] = {};
    long long ph_t = clock64();
#define PLBM_PHASE(k)                  \
    {                                  \
        const long long t_ = clock64(); \
        ph_acc[k] += t_ - ph_t;        \
        ph_t = t_;                     \
    }
#else
#define PLBM_PHASE(k)
#endif
    fill_zghost(-1);
#pragma unroll 1
    for (int p = 0; p < LAG; ++p) {
        issue_pulls(p);
        issue_ring(p);
        cp_async_commit();
        expect(p);
        cp_async_wait<0>();
        __syncthreads();
        psi_pass(p);
    }
    issue_pulls(LAG);
    cp_async_commit();
    __syncthreads();
    issue_ring(LAG);
    cp_async_commit();
    if (warp == 0)
        for (int p = 0; p < LAG; ++p) wait_pushed(p);
    __syncthreads();
#pragma unroll 1
    for (int z = 0; z < E; ++z) {
        const int pn = z + LAG;
        if (pn < E) {
            expect(pn);
            cp_async_wait<0>();  // pulls and ghost ring of plane pn have landed
            PLBM_PHASE(0)
            psi_pass(pn);
            PLBM_PHASE(1)
            issue_pulls(pn + 1);  // this thread's landing slots were just read
            cp_async_commit();
            PLBM_PHASE(2)
        } else if (pn == E) {
            fill_zghost(E);
        }
        double f[Q], rho, u0, u1, u2;
        if constexpr (EARLY) collide_head(z, f, rho, u0, u1, u2);
        PLBM_PHASE(3)
        // The peers' psi of plane z+1: one warp polls the mbarrier, the CTA
        // barrier then releases the others (they wait in bar.sync instead of
        // spinning) and carries the acquired data to them.
        if (warp == POLL_WARP && z + 1 < E && z + 1 >= LAG) wait_pushed(z + 1);
        PLBM_PHASE(4)
        __syncthreads();  // psi plane pn visible; every warp is past collide(z-1)
        PLBM_PHASE(5)
        flush_xcol(z - 1);
        issue_ring(pn + 1);  // its ring slot is no longer read by anyone
        cp_async_commit();
        PLBM_PHASE(6)
        if constexpr (!EARLY) collide_head(z, f, rho, u0, u1, u2);
        collide_plane(z, f, rho, u0, u1, u2);
        PLBM_PHASE(7)
    }
#ifdef PLBM_PHASES
    if (d.probe && (tid & 31) == 0)
        for (int k = 0; k < 8; ++k) atomicAdd(&d.probe[warp * 8 + k], ph_acc[k]);
#endif
#undef PLBM_PHASE
    {
        const unsigned m1 = __reduce_add_sync(0xffffffffu, negs);
        const unsigned m2 = __reduce_add_sync(0xffffffffu, clamps);
        const unsigned m3 = __reduce_add_sync(0xffffffffu, zero_rho);
        const bool sus = __any_sync(0xffffffffu, suspect);
        if ((tid & 31) == 0) {
            if (m1) atomicAdd(&d.cnt[CNT_NEG], (unsigned long long)m1);
            if (m2) atomicAdd(&d.cnt[CNT_CLAMP], (unsigned long long)m2);
            if (m3) atomicAdd(&d.cnt[CNT_ZERO_RHO], (unsigned long long)m3);
            if (sus) {
                d.suspect[slot] = 1;
                if (d.susp_any) atomicOr(&d.susp_any[iter & 1], 1u);
            }
        }
    }
    cp_async_wait<0>();
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    const bool fused = (d.face_flags & FACE_FUSED) != 0;
    __syncthreads();
    flush_xcol(E - 1);
    if (fused) __threadfence();  // this thread's f_post / u_face / xcol stores, GPU-wide
    __syncthreads();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(s_tmem),
                     "n"(T::NCOLS));
    auto cluster_sync = [&] {
        if constexpr (T::CL > 1) {
            asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
            asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
        } else {
            __syncthreads();
        }
    };
    cluster_sync();  // every push into a peer has landed; the whole tile is written
#ifndef PLBM_PHASES
    if (d.probe && tid == 0) {
        d.probe[3 * blockIdx.x] = smid();
        d.probe[3 * blockIdx.x + 1] = t_start;
        d.probe[3 * blockIdx.x + 2] = global_ns();
    }
#endif
    if (NH != 1 || !fused) return;  // (the fused face pass needs whole-tile clusters)

    // ---- fused face pass ---------------------------------------------------------
    // This tile is complete: count it towards itself and its active geometric
    // neighbours.  Whoever brings a tile's count to dep_need (all of the tiles
    // its face cells pull from are written) runs that tile's face pass: psi
    // faces for the next step, criterion, P5 NaN check.  Nobody waits.
    if (rank == 0 && tid == 0) {
        int n = 0;
        auto count = [&](int m) {
            if (atomicAdd(&d.dep_cnt[m], 1) == d.dep_need[m] - 1) {
                d.dep_cnt[m] = 0;  // every count of this step is in: reset for the next
                s_ready[n++] = m;
            }
        };
        count(slot);
        for (int k = 0; k < 18; ++k) {
            const int m = d.geo[size_t(slot) * 18 + k];
            if (m >= 0) count(m);
        }
        s_nready = n;
        __threadfence();  // acquire side of the counts: the other tiles' stores
    }
    cluster_sync();
    int ready[20];
    int nready;
    {
        uint32_t a0;
        asm volatile("mapa.shared::cluster.u32 %0, %1, 0;\n" : "=r"(a0) : "r"(smem_u32(&s_nready)));
        asm volatile("ld.shared::cluster.u32 %0, [%1];\n" : "=r"(nready) : "r"(a0) : "memory");
        asm volatile("mapa.shared::cluster.u32 %0, %1, 0;\n" : "=r"(a0) : "r"(smem_u32(&s_ready[0])));
        for (int j = 0; j < nready; ++j)
            asm volatile("ld.shared::cluster.u32 %0, [%1];\n" : "=r"(ready[j]) : "r"(a0 + 4u * j) : "memory");
    }
    cluster_sync();  // rank 0 may exit once everyone has the list
    const int per = (6 + d.mid_faces) * E2 / T::NB;
    for (int j = 0; j < nready; ++j)
        face_pass_part<E, NT>(d, ready[j], c, 1, yb * per, (yb + 1) * per, src_buf ^ 1, iter, rt_pull,
                              s_solid, s_tc);
}

}  // namespace plbm
