// dispatch.cuh — the per-(E, C, psi) table of step-loop kernels.
//
// The kernels are instantiated in one translation unit per tile extent
// (inst_e8.cu .. inst_e64.cu, compiled in parallel); each unit has its own
// copy of the constants P (kernels.cuh), uploaded through set_params.
#pragma once

#include "kernels.cuh"

namespace plbm {

using MainFn = void (*)(Dev, const int*, int, int, long, unsigned, cudaStream_t);
struct Kernels {
    MainFn main_plain;  // variant 1 (and the only kernel for E = 8 / psi-free)
    MainFn main_pc;     // variant 0: one CTA per (block, component), cp.async staged
    MainFn main_pc_late;  // variant 21: the collision head after the cluster wait
    MainFn main_pc_mem;   // variant 24 (PLBM_PROBES builds only): memory-only probe (E = 32, C = 2)
    MainFn main_pc2;    // variant 22: psi computed two planes ahead
    MainFn main_aa[2];  // A-A storage: AA_LOCAL / AA_NEIGH steps (k_main_pc, else the whole-tile plain kernel)
    MainFn main_pc_split[2];     // k_main_pc with 2 / 4 clusters per tile (E >= 32; see Engine::set_variant)
    MainFn main_aa_split[2][2];  // the same for the A-A steps [split][AA_LOCAL / AA_NEIGH]
    int nhmax = 1;               // finest split: the face pass writes its boundary rows (Dev::mid_faces)
    bool aa_xcol = false;  // the A-A kernels write the xcol side buffers (k_main_pc does)
    void (*face)(Dev, const int*, int, int, long, unsigned, cudaStream_t);
    void (*face_v[2])(Dev, const int*, int, int, long, unsigned, cudaStream_t);
    void (*p5)(Dev, const int*, int, long, unsigned, cudaStream_t);
    void (*readback)(Dev, int, int, int, double*, int, cudaStream_t);
    void (*gather)(Dev, const int*, int, int, int, int, double*, int, int, int, cudaStream_t);
    void (*preload)();  // loads every kernel of this (E, C) (see Engine::init: lazy loading)
    void (*set_params)(const Params&, cudaStream_t);  // this unit's copy of the constants P
    int nt;
};

Kernels pick_kernels_e8(int C, bool nopsi);
Kernels pick_kernels_e16(int C, bool nopsi);
Kernels pick_kernels_e32(int C, bool nopsi);
Kernels pick_kernels_e64(int C, bool nopsi);

}  // namespace plbm
