// physics.cuh — per-cell building blocks of the fused step kernels (sm_100a):
// the TMEM stash of a cell's 19 populations + rho (tcgen05.st / tcgen05.ld,
// 32x32b shape, one TMEM lane per thread), the Shan-Chen neighbour sums, the
// BGK collision with velocity-shift forcing, and the velocity of a pulled cell.
// Every expression restates the reference's tree exactly (see lattice.cuh).
#pragma once

#include "kernels.cuh"

namespace plbm {

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

// One component's BGK collision with the velocity-shift forcing
// (engine.cpp:450-475) given the total force F.  f is overwritten with the
// post-collision populations, each stored through out(i, value) (StoreF:
// A-B or A-A placement); xc (x-column lanes only, else nullptr) receives a
// copy of all 19 at stride xstride.  `suspect` is set when a stored value
// leaves the P5 screen's range (lattice.cuh Screen).
template <class St>
__device__ __forceinline__ void collide_bgk(double* f, double rho, double u0, double u1,
                                            double u2, double F0, double F1, double F2,
                                            double om, const St& out,
                                            unsigned& zero_rho, int& suspect, double* xc = nullptr,
                                            int xstride = 0) {

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
        out(I, f[I]);                                                                        \
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
        out(I, f[I]);                                                                        \
    }
        PLBM_TM_FORCED(0) PLBM_TM_FORCED(1) PLBM_TM_FORCED(2) PLBM_TM_FORCED(3)
        PLBM_TM_FORCED(4) PLBM_TM_FORCED(5) PLBM_TM_FORCED(6) PLBM_TM_FORCED(7)
        PLBM_TM_FORCED(8) PLBM_TM_FORCED(9) PLBM_TM_FORCED(10) PLBM_TM_FORCED(11)
        PLBM_TM_FORCED(12) PLBM_TM_FORCED(13) PLBM_TM_FORCED(14) PLBM_TM_FORCED(15)
        PLBM_TM_FORCED(16) PLBM_TM_FORCED(17) PLBM_TM_FORCED(18)
#undef PLBM_TM_FORCED
    }
    {
        Screen sc;
#pragma unroll
        for (int i = 0; i + 1 < Q; i += 2) sc.add2(f[i], f[i + 1]);
        sc.add(f[Q - 1]);
        suspect |= sc.suspect();
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

}  // namespace plbm
