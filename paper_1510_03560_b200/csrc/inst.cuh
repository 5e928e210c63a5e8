// inst.cuh — instantiation of the step-loop kernels for one tile extent E
// (included by inst_e<E>.cu; see dispatch.cuh).
#pragma once

#include "kernels.cuh"
#include "kernels_pc.cuh"
#include "dispatch.cuh"

#include <cuda_runtime.h>

#include <stdexcept>

namespace plbm {
namespace {

// which (E, C) run k_main_pc, and its CTA size
template <int E>
struct PcNT {
    static constexpr int value = E == 64 ? 512 : 256;
};
template <int E, int C, bool NOPSI>
struct HasPc {
    static constexpr bool value = !NOPSI && (E == 16 || E == 32 || (E == 64 && C <= 2));
};

// split-tile clusters (NH = 2 and the finest split, nh_fine: 4 clusters per
// tile at E = 32, 8 at E = 64 — one y-block x C components each) for
// E >= 32; the face pass writes the boundary rows of the finest split
template <int E, int C, bool NOPSI>
struct HasHalf {
    static constexpr bool value = !NOPSI && (E == 32 || E == 64);
};
#ifndef PLBM_E64_NH
#define PLBM_E64_NH 8  // the finest split at E = 64: one y-block per cluster (4: two, measured slower at C >= 2)
#endif
template <int E>
constexpr int nh_fine() { return E == 64 ? PLBM_E64_NH : 4; }
// experiment builds (build.py --exp): the split kernel's pipeline shape
#ifndef PLBM_SPLIT_LAG
#define PLBM_SPLIT_LAG 1
#endif
#ifndef PLBM_SPLIT_EARLY
#define PLBM_SPLIT_EARLY true
#endif

template <int E, int C, int LAG, int NT = 256, bool EARLY = true, bool MEMONLY = false, int AA = AA_OFF,
          int NH = 1>
void launch_pc(Dev d, const int* act, int src, int wu, long it, unsigned ntiles, cudaStream_t s) {
    using T = PcCfg<E, C, LAG, NT, NH>;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(ntiles * NH * T::CL);
    cfg.blockDim = dim3(T::NT);
    cfg.dynamicSmemBytes = T::SMEM;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = T::CL;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, k_main_pc<E, C, LAG, NT, EARLY, MEMONLY, AA, NH>, d, act, src, wu, it);
}

template <int E, int C, bool NOPSI>
Kernels make_kernels() {
    constexpr int NT = E * E < 256 ? E * E : 256;
    constexpr int BZ = E < 8 ? E : 8;
    constexpr int YB = E == 64 ? 16 : E;  // y-chunk of the plain kernel (E = 64: psi ring in smem)
    constexpr int G = E + 2;
    constexpr size_t SMEM_PLAIN = NOPSI ? 0 : size_t(3) * C * G * (YB + 2) * sizeof(double);
    Kernels k;
    k.nt = NT;
    // (static shared memory counts against the same 48 KB default: opt in
    // whenever there is a dynamic ring)
    if (SMEM_PLAIN > 0)
        cudaFuncSetAttribute(k_main<E, C, BZ, NT, NOPSI, YB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             int(SMEM_PLAIN));
    k.main_plain = [](Dev d, const int* act, int src, int wu, long it, unsigned ntiles, cudaStream_t s) {
        k_main<E, C, BZ, NT, NOPSI, YB><<<ntiles * (E / BZ) * (E / YB), NT, SMEM_PLAIN, s>>>(d, act, src, wu, it);
    };
    k.main_pc = k.main_pc2 = k.main_pc_late = k.main_pc_mem = nullptr;
    k.main_aa[0] = k.main_aa[1] = nullptr;
    for (int j = 0; j < 2; ++j) k.main_pc_split[j] = k.main_aa_split[j][0] = k.main_aa_split[j][1] = nullptr;
    k.nhmax = HasHalf<E, C, NOPSI>::value ? nh_fine<E>() : 1;
    // k_main_pc: 256-thread CTAs (8 warps, 2 per SM) for E = 16 / 32; for
    // E = 64 one 512-thread CTA per SM (8 rows of 64 cells, 16 warps) so that
    // a tile is 8 y-blocks x C components: a 16-CTA cluster at C = 2
    constexpr int PNT = PcNT<E>::value;
    auto setup = [](auto fn, int smem, int cl) {
        cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (cl > 8) cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    };
    // split-tile clusters (E = 64 at C = 3 too: 12 / 6 CTAs where a whole
    // tile would need 24)
    if constexpr (HasHalf<E, C, NOPSI>::value) {
        using TH = PcCfg<E, C, 1, PNT, 2>;
        using TQ = PcCfg<E, C, 1, PNT, nh_fine<E>()>;
        using TX = PcCfg<E, C, PLBM_SPLIT_LAG, PNT, nh_fine<E>()>;
        setup(k_main_pc<E, C, 1, PNT, true, false, AA_OFF, 2>, TH::SMEM, TH::CL);
        setup(k_main_pc<E, C, PLBM_SPLIT_LAG, PNT, PLBM_SPLIT_EARLY, false, AA_OFF, nh_fine<E>()>, TX::SMEM, TX::CL);
        k.main_pc_split[0] = launch_pc<E, C, 1, PNT, true, false, AA_OFF, 2>;
        k.main_pc_split[1] = launch_pc<E, C, PLBM_SPLIT_LAG, PNT, PLBM_SPLIT_EARLY, false, AA_OFF, nh_fine<E>()>;
#ifndef PLBM_NO_AA
        setup(k_main_pc<E, C, 1, PNT, true, false, AA_LOCAL, 2>, TH::SMEM, TH::CL);
        setup(k_main_pc<E, C, 1, PNT, true, false, AA_NEIGH, 2>, TH::SMEM, TH::CL);
        setup(k_main_pc<E, C, 1, PNT, true, false, AA_LOCAL, nh_fine<E>()>, TQ::SMEM, TQ::CL);
        setup(k_main_pc<E, C, 1, PNT, true, false, AA_NEIGH, nh_fine<E>()>, TQ::SMEM, TQ::CL);
        k.main_aa_split[0][0] = launch_pc<E, C, 1, PNT, true, false, AA_LOCAL, 2>;
        k.main_aa_split[0][1] = launch_pc<E, C, 1, PNT, true, false, AA_NEIGH, 2>;
        k.main_aa_split[1][0] = launch_pc<E, C, 1, PNT, true, false, AA_LOCAL, nh_fine<E>()>;
        k.main_aa_split[1][1] = launch_pc<E, C, 1, PNT, true, false, AA_NEIGH, nh_fine<E>()>;
        k.aa_xcol = true;
#endif
    }
    if constexpr (HasPc<E, C, NOPSI>::value) {
        using T1 = PcCfg<E, C, 1, PNT>;
        setup(k_main_pc<E, C, 1, PNT>, T1::SMEM, T1::CL);
        k.main_pc = launch_pc<E, C, 1, PNT>;
        setup(k_main_pc<E, C, 1, PNT, false>, T1::SMEM, T1::CL);
        k.main_pc_late = launch_pc<E, C, 1, PNT, false>;
#ifdef PLBM_PROBES
        if constexpr (E == 32 && C == 2) {
            setup(k_main_pc<E, C, 1, 256, true, true>, T1::SMEM, T1::CL);
            k.main_pc_mem = launch_pc<E, C, 1, 256, true, true>;
        }
#endif
        if constexpr (C <= 2) {
            using T2 = PcCfg<E, C, 2, PNT>;
            setup(k_main_pc<E, C, 2, PNT>, T2::SMEM, T2::CL);
            k.main_pc2 = launch_pc<E, C, 2, PNT>;
        }
#ifndef PLBM_NO_AA
        setup(k_main_pc<E, C, 1, PNT, true, false, AA_LOCAL>, T1::SMEM, T1::CL);
        setup(k_main_pc<E, C, 1, PNT, true, false, AA_NEIGH>, T1::SMEM, T1::CL);
        k.main_aa[0] = launch_pc<E, C, 1, PNT, true, false, AA_LOCAL>;
        k.main_aa[1] = launch_pc<E, C, 1, PNT, true, false, AA_NEIGH>;
        k.aa_xcol = true;
#endif
    } else if constexpr (E <= 32) {
#ifndef PLBM_NO_AA
        // A-A with the plain kernel: one CTA per tile (no recomputed halos)
        constexpr size_t SMEM_AA = NOPSI ? 0 : size_t(3) * C * G * G * sizeof(double);
        if (SMEM_AA > 0) {
            cudaFuncSetAttribute(k_main<E, C, E, NT, NOPSI, E, AA_LOCAL>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, int(SMEM_AA));
            cudaFuncSetAttribute(k_main<E, C, E, NT, NOPSI, E, AA_NEIGH>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, int(SMEM_AA));
        }
        k.main_aa[0] = [](Dev d, const int* act, int src, int wu, long it, unsigned ntiles, cudaStream_t s) {
            k_main<E, C, E, NT, NOPSI, E, AA_LOCAL><<<ntiles, NT, SMEM_AA, s>>>(d, act, src, wu, it);
        };
        k.main_aa[1] = [](Dev d, const int* act, int src, int wu, long it, unsigned ntiles, cudaStream_t s) {
            k_main<E, C, E, NT, NOPSI, E, AA_NEIGH><<<ntiles, NT, SMEM_AA, s>>>(d, act, src, wu, it);
        };
#endif
    }
    // k_face at 4 CTAs/SM, one item in flight per thread (64 registers),
    // measured faster than 2 CTAs/SM with a one-item prefetch (PLBM_FACE_VARIANT=1)
    k.face_v[0] = [](Dev d, const int* act, int src, int flags, long it, unsigned ntiles, cudaStream_t s) {
        k_face<E, C, NT, 4, false><<<ntiles * (6 + d.mid_faces), NT, 0, s>>>(d, act, src, flags, it);
    };
    k.face_v[1] = [](Dev d, const int* act, int src, int flags, long it, unsigned ntiles, cudaStream_t s) {
        k_face<E, C, NT, 2, true><<<ntiles * (6 + d.mid_faces), NT, 0, s>>>(d, act, src, flags, it);
    };
    k.face = k.face_v[0];
    k.p5 = [](Dev d, const int* act, int src, long it, unsigned ntiles, cudaStream_t s) {
        k_p5<E, C, 256><<<ntiles, 256, 0, s>>>(d, act, src, it);
    };
    // CUDA loads a kernel lazily at its first launch, and loading may wait
    // for the device: a rank whose first launch of some kernel happens while
    // its peer's rank-barrier kernel spins would deadlock.  Load them all now.
    k.preload = [] {
        cudaFuncAttributes a;
        auto ld = [&](const void* f) { cudaFuncGetAttributes(&a, f); };
        ld((const void*)k_main<E, C, BZ, NT, NOPSI, YB>);
        ld((const void*)k_face<E, C, NT, 4, false>);
        ld((const void*)k_face<E, C, NT, 2, true>);
        ld((const void*)k_p5<E, C, 256>);
        ld((const void*)k_readback<E>);
        ld((const void*)k_gather<E>);
        if constexpr (E <= 32) {
            ld((const void*)k_main<E, C, E, NT, NOPSI, E, AA_LOCAL>);
            ld((const void*)k_main<E, C, E, NT, NOPSI, E, AA_NEIGH>);
        }
        if constexpr (HasPc<E, C, NOPSI>::value) {
            constexpr int PN = PcNT<E>::value;
            ld((const void*)k_main_pc<E, C, 1, PN>);
            ld((const void*)k_main_pc<E, C, 1, PN, false>);
            ld((const void*)k_main_pc<E, C, 1, PN, true, false, AA_LOCAL>);
            ld((const void*)k_main_pc<E, C, 1, PN, true, false, AA_NEIGH>);
            if constexpr (C <= 2) ld((const void*)k_main_pc<E, C, 2, PN>);
        }
        if constexpr (HasHalf<E, C, NOPSI>::value) {
            constexpr int PN = PcNT<E>::value;
            ld((const void*)k_main_pc<E, C, 1, PN, true, false, AA_OFF, 2>);
            ld((const void*)k_main_pc<E, C, 1, PN, true, false, AA_LOCAL, 2>);
            ld((const void*)k_main_pc<E, C, 1, PN, true, false, AA_NEIGH, 2>);
            ld((const void*)k_main_pc<E, C, PLBM_SPLIT_LAG, PN, PLBM_SPLIT_EARLY, false, AA_OFF, nh_fine<E>()>);
            ld((const void*)k_main_pc<E, C, 1, PN, true, false, AA_LOCAL, nh_fine<E>()>);
            ld((const void*)k_main_pc<E, C, 1, PN, true, false, AA_NEIGH, nh_fine<E>()>);
        }
    };
    k.set_params = [](const Params& p, cudaStream_t s) {
        cudaMemcpyToSymbolAsync(P, &p, sizeof(Params), 0, cudaMemcpyHostToDevice, s);
    };
    k.readback = [](Dev d, int slot, int c, int src, double* out, int skind, cudaStream_t s) {
        k_readback<E><<<(E * E * E + 255) / 256, 256, 0, s>>>(d, slot, c, src, out, skind);
    };
    k.gather = [](Dev d, const int* act, int ntiles, int kind, int c, int src, double* grid, int D0, int D1,
                  int skind, cudaStream_t s) {
        k_gather<E><<<dim3((E * E * E + 255) / 256, ntiles), 256, 0, s>>>(d, act, kind, c, src, grid, D0, D1,
                                                                          skind);
    };
    return k;
}

template <int E>
Kernels pick_c(int C, bool nopsi) {
#ifdef PLBM_ONLY_E32C2  // experiment builds: the bench instantiation only (fast compile)
    if (E == 32 && C == 2 && !nopsi) return make_kernels<32, 2, false>();
    throw std::invalid_argument("PLBM_ONLY_E32C2 build: E = 32, C = 2 only");
#else
    switch (C) {
    case 1: return nopsi ? make_kernels<E, 1, true>() : make_kernels<E, 1, false>();
    case 2: return nopsi ? make_kernels<E, 2, true>() : make_kernels<E, 2, false>();
    case 3: return nopsi ? make_kernels<E, 3, true>() : make_kernels<E, 3, false>();
    default: throw std::invalid_argument("n_components must be 1..3 on the GPU path");
    }
#endif
}

}  // namespace
}  // namespace plbm

#define PLBM_INSTANTIATE(E_)                                                              \
    namespace plbm {                                                                      \
    Kernels pick_kernels_e##E_(int C, bool nopsi) { return pick_c<E_>(C, nopsi); }       \
    }
