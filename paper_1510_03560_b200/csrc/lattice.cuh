// lattice.cuh — D3Q19 lattice + multiphase closure as sm_100a device code.
//
// Every function reproduces the reference's floating-point expression tree
// exactly (the translation unit is compiled with -fmad=false, so nvcc never
// contracts a multiply-add), which is what makes the B200 engine bit-identical
// to the CPU reference in FP64.  Algebraic shortcuts are used only where they
// are provably bit-neutral:
//   * e_i components are in {-1,0,+1}: a product with 0 contributes a signed
//     zero that can never change a non-zero running sum, and a product with
//     +-1 is exact, so those terms are folded at compile time;
//   * opposite velocity pairs share |e.u| and (e.u)^2 exactly (IEEE rounding
//     is sign-symmetric), so each pair evaluates the quadratic term once;
//   * ideal-like EOS (a = b = 0) reduces pr_pressure to (rho R) T exactly.
// The reference expression each function restates is cited inline.
#pragma once

#include <cstdint>

#include "ieee_div.cuh"

namespace plbm {

constexpr int Q = 19;

// proj/src/stencil.cpp:21-34 — velocity order (part of the parity contract).
__host__ __device__ constexpr int ex_(int i) {
    constexpr int t[Q] = {0, 1, -1, 0, 0, 0, 0, 1, -1, 1, -1, 1, -1, 1, -1, 0, 0, 0, 0};
    return t[i];
}
__host__ __device__ constexpr int ey_(int i) {
    constexpr int t[Q] = {0, 0, 0, 1, -1, 0, 0, 1, -1, -1, 1, 0, 0, 0, 0, 1, -1, 1, -1};
    return t[i];
}
__host__ __device__ constexpr int ez_(int i) {
    constexpr int t[Q] = {0, 0, 0, 0, 0, 1, -1, 0, 0, 0, 0, 1, -1, -1, 1, 1, -1, -1, 1};
    return t[i];
}
// proj/src/stencil.cpp:57-69 (derived opposite map).
__host__ __device__ constexpr int opp_(int i) {
    constexpr int t[Q] = {0, 2, 1, 4, 3, 6, 5, 8, 7, 10, 9, 12, 11, 14, 13, 16, 15, 18, 17};
    return t[i];
}
// x-column side buffer ("xcol"): the fused kernel also stores the post-
// collision populations of the four x-boundary columns (x = 0, 1, E-2, E-1)
// that the x faces' pulls need, y-contiguous, so the face pass reads them
// coalesced instead of one 8-byte element per 32-byte sector of the SoA block.
//   class 0 (x = 0):   e_x in {0, -1} (own x = 0 face, -x neighbour's x = E-1 face)
//   class 1 (x = 1):   e_x = -1       (own x = 0 face)
//   class 2 (x = E-2): e_x = +1       (own x = E-1 face)
//   class 3 (x = E-1): e_x in {0, +1} (own x = E-1 face, +x neighbour's x = 0 face)
constexpr int XN = 38;  // (class, direction) pairs per component
__host__ __device__ constexpr int xslot_(int cls, int i) {
    constexpr int t[4][Q] = {
        {0, -1, 1, 2, 3, 4, 5, -1, 6, -1, 7, -1, 8, -1, 9, 10, 11, 12, 13},
        {-1, -1, 14, -1, -1, -1, -1, -1, 15, -1, 16, -1, 17, -1, 18, -1, -1, -1, -1},
        {-1, 19, -1, -1, -1, -1, -1, 20, -1, 21, -1, 22, -1, 23, -1, -1, -1, -1, -1},
        {24, 25, -1, 26, 27, 28, 29, 30, -1, 31, -1, 32, -1, 33, -1, 34, 35, 36, 37}};
    return t[cls][i];
}
// inverse map: xcol slot -> (class, direction)
__host__ __device__ constexpr int xslot_cls(int s) { return s < 14 ? 0 : s < 19 ? 1 : s < 24 ? 2 : 3; }
__host__ __device__ constexpr int xslot_dir(int s) {
    constexpr int t[XN] = {0, 2, 3, 4, 5, 6, 8, 10, 12, 14, 15, 16, 17, 18, 2, 8, 10, 12, 14,
                           1, 7, 9, 11, 13, 0, 1, 3, 4, 5, 6, 7, 9, 11, 13, 15, 16, 17, 18};
    return t[s];
}
// xslot_ with a compile-time direction and a runtime class, without a table
// in local memory
__host__ __device__ __forceinline__ constexpr int xslot_sel(int cls, int i) {
    return cls == 0 ? xslot_(0, i) : cls == 1 ? xslot_(1, i) : cls == 2 ? xslot_(2, i) : xslot_(3, i);
}

// weight class: 0 -> 1/3, 1 -> 1/18, 2 -> 1/36
__host__ __device__ constexpr int wclass_(int i) { return i == 0 ? 0 : (i <= 6 ? 1 : 2); }

#define PLBM_W0 (1.0 / 3.0)
#define PLBM_W1 (1.0 / 18.0)
#define PLBM_W2 (1.0 / 36.0)
#define PLBM_CS2 (1.0 / 3.0)

__host__ __device__ constexpr double w_(int i) {
    return i == 0 ? PLBM_W0 : (i <= 6 ? PLBM_W1 : PLBM_W2);
}

// Per-component constants (host-precomputed with the same IEEE operations
// as the reference computes them per call).
struct CompConst {
    double omega;        // 1.0 / tau                    (engine.cpp:419)
    double gravity[3];
    int has_gravity;     // engine.cpp:416-418
    int psi_free;        // a=b=0, R=1, T=cs2  =>  psi == +-0 everywhere
    int ideal;           // a == 0 && b == 0
    int pad;
    double R, T, b;      // EOS
    double a_theta;      // a * theta                    (physics.cpp:22-24)
    double two_b, b_b;   // 2b, b*b                      (physics.cpp:25)
    double cs2_g;        // cs2 * g_self                 (physics.cpp:36)
    double c1f;          // -beta * g_self               (physics.cpp:59)
    double c2;           // -0.5 * (1 - beta) * g_self   (physics.cpp:60)
    double rho_amb, psi_amb, psi_nb; // ambient rho/psi; psi of a newborn cell
    double feq_amb[Q];   // equilibrium at rest          (tilemap.cpp:13-28)
};

// proj/include/plbm/kernels.hpp:17-28 — f_eq(rho, u) for all 19 directions.
// out_i = (w_i rho) * (((1 + eu*3) + ((0.5 eu) eu * 3) * 3) - (0.5 uu) * 3)
__device__ __forceinline__ void equilibrium(double rho, double u0, double u1, double u2,
                                            double* out) {
    const double uu = u0 * u0 + u1 * u1 + u2 * u2;
    const double t3 = (0.5 * uu) * 3.0;
    const double wr0 = PLBM_W0 * rho, wr1 = PLBM_W1 * rho, wr2 = PLBM_W2 * rho;
    out[0] = wr0 * (1.0 - t3);  // eu = +-0 for the rest vector
    // + members of the 9 opposite pairs: 1,3,5,7,9,11,13,15,17
    const double eus[9] = {u0, u1, u2, u0 + u1, u0 - u1, u0 + u2, u0 - u2, u1 + u2, u1 - u2};
#pragma unroll
    for (int p = 0; p < 9; ++p) {
        const double eu = eus[p];
        const double a = eu * 3.0;
        const double b = (((0.5 * eu) * eu) * 3.0) * 3.0;
        const double wr = p < 3 ? wr1 : wr2;
        out[1 + 2 * p] = wr * (((1.0 + a) + b) - t3);
        out[2 + 2 * p] = wr * (((1.0 - a) + b) - t3);
    }
}

// Single-direction equilibrium, same tree as above (used on the fly).
template <int I>
__device__ __forceinline__ double feq_dir(double wr, double eu, double t3) {
    if constexpr (I == 0) {
        return wr * (1.0 - t3);
    } else {
        const double a = eu * 3.0;
        const double b = (((0.5 * eu) * eu) * 3.0) * 3.0;
        return (I & 1) ? wr * (((1.0 + a) + b) - t3) : wr * (((1.0 - a) + b) - t3);
    }
}

// e_i . u for the "+" member of direction I's pair (exact; see header).
template <int I>
__device__ __forceinline__ double eu_pair(double u0, double u1, double u2) {
    constexpr int p = (I - 1) / 2;
    if constexpr (p == 0) return u0;
    else if constexpr (p == 1) return u1;
    else if constexpr (p == 2) return u2;
    else if constexpr (p == 3) return u0 + u1;
    else if constexpr (p == 4) return u0 - u1;
    else if constexpr (p == 5) return u0 + u2;
    else if constexpr (p == 6) return u0 - u2;
    else if constexpr (p == 7) return u1 + u2;
    else return u1 - u2;
}

// proj/include/plbm/kernels.hpp:31-48 — rho and momentum by sequential sums
// (i order); zero-e terms are exact no-ops on a running sum that starts at +0.
__device__ __forceinline__ void moments(const double* f, double& rho, double& u0, double& u1,
                                        double& u2) {
    double r = 0.0;
#pragma unroll
    for (int i = 0; i < Q; ++i) r += f[i];
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
        u0 = m0 / r;
        u1 = m1 / r;
        u2 = m2 / r;
    } else {
        u0 = u1 = u2 = 0.0;
    }
    rho = r;
}

__device__ __forceinline__ double sum19(const double* f) {
    double r = 0.0;
#pragma unroll
    for (int i = 0; i < Q; ++i) r += f[i];
    return r;
}

// proj/src/physics.cpp:12-27; returns false at the b*rho >= 1 pole.
__device__ __forceinline__ bool pr_pressure(double rho, const CompConst& k, double& p) {
    if (k.ideal) {  // a = b = 0: ideal/(1-0) - 0/(1+0-0) == (rho R) T exactly
        p = (rho * k.R) * k.T;
        return true;
    }
    if (k.b * rho >= 1.0) return false;
    // ideal = ((rho R) T) / (1 - b rho); attr = ((a theta rho) rho) / ((1 + 2b rho) - (b^2 rho) rho)
    const double n1 = (rho * k.R) * k.T, d1 = 1.0 - k.b * rho;
    const double n2 = (k.a_theta * rho) * rho, d2 = (1.0 + k.two_b * rho) - (k.b_b * rho) * rho;
    bool ok = true;
    double ideal = div_nv(n1, d1, rcp_nv(d1), ok);
    double attr = div_nv(n2, d2, rcp_nv(d2), ok);
    if (!ok) {
        ideal = n1 / d1;
        attr = n2 / d2;
    }
    p = ideal - attr;
    return true;
}

// proj/src/physics.cpp:34-42; *clamped set on a negative radicand.
__device__ __forceinline__ double pseudo_potential(double rho, double press, const CompConst& k,
                                                   bool& clamped) {
    const double num = 2.0 * (press - PLBM_CS2 * rho);
    bool ok = true;
    double radicand = div_nv(num, k.cs2_g, rcp_nv(k.cs2_g), ok);
    if (!ok) radicand = num / k.cs2_g;
    if (radicand < 0.0) {
        clamped = true;
        return 0.0;
    }
    clamped = false;
    return sqrt(radicand);
}

// P5 screen (proj/src/engine.cpp:500-512 checks rho and u of every post-stream
// cell for non-finite values).  Claim: if every population a cell pulls is 0 or
// has 2^-400 <= |f| < 2^400, its moments are finite.  Every such value is a
// multiple of 2^-452, so every partial sum of rho (and m) is an exact multiple
// of 2^-452 (a rounded sum of multiples stays a multiple), hence rho == 0 (u =
// 0 by moments' rule) or |rho| >= 2^-452; with |m| < 19 * 2^400 < 2^405 the
// quotient |u| <= 2^857 is finite.  The fused kernels therefore track the
// exponent range of every stored post-collision value; a tile whose values
// leave [2^-400, 2^400) (exact zeros included, conservatively) is marked
// suspect and k_p5 checks its post-stream moments exactly.  The ambient
// populations (the other pulled source) are checked once on the host.
constexpr uint32_t SCREEN_LO = 623u << 20;   // |hi word| of 2^-400
constexpr uint32_t SCREEN_HI = 1423u << 20;  // |hi word| of 2^400
struct Screen {
    // (|hi| << 1) - (LO << 1) wraps for values below the range, so one unsigned
    // max over the 19 values covers both ends: suspect iff max >= 2 (HI - LO)
    uint32_t mx = 0u;
    __device__ __forceinline__ static uint32_t key(double a) {
        return (uint32_t(__double2hiint(a)) << 1) - (SCREEN_LO << 1);
    }
    __device__ __forceinline__ void add2(double a, double b) { mx = __vimax3_u32(mx, key(a), key(b)); }
    __device__ __forceinline__ void add(double a) { mx = max(mx, key(a)); }
    __device__ __forceinline__ bool suspect() const { return mx >= ((SCREEN_HI - SCREEN_LO) << 1); }
};
__host__ __device__ inline bool screen_ok(double v) {
    if (v == 0.0) return true;
    const double a = v < 0 ? -v : v;
    return a >= 0x1p-400 && a < 0x1p400;
}

}  // namespace plbm
