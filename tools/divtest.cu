// divtest.cu — bit-for-bit check of div_nv (csrc/ieee_div.cuh) against the
// '/' operator on sm_100a, over random operands spanning the whole exponent
// range plus special values.  Prints the mismatch count; exit code 1 if any.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -I paper_1510_03560_b200/csrc
//      -o build/divtest tools/divtest.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#include "ieee_div.cuh"

__device__ uint64_t mix(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

__device__ double pick(uint64_t h, int mode) {
    if (mode == 0) return __longlong_as_double((long long)h);  // any bit pattern
    // moderate exponents around the LBM value range, random mantissa and sign
    const uint64_t exp = 1023 - 40 + (h >> 56) % 80;
    return __longlong_as_double((long long)((h & 0x800FFFFFFFFFFFFFull) | (exp << 52)));
}

// mine and the stock operator in separate launches so nothing is shared
__global__ void k_mine(uint64_t n, uint64_t seed, int mode, double* out, unsigned char* fast) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x) {
        const double b = pick(mix(seed ^ (2 * i)), mode);
        const double a0 = pick(mix(seed ^ (2 * i + 1)), mode);
        const double a1 = pick(mix(seed ^ (2 * i + 1) ^ 0x5555), mode);
        bool ok = true;
        const double r = plbm::rcp_nv(b);
        out[2 * i] = plbm::div_nv(a0, b, r, ok);
        out[2 * i + 1] = plbm::div_nv(a1, b, r, ok);
        fast[i] = ok;
    }
}
__global__ void k_stock(uint64_t n, uint64_t seed, int mode, double* out) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x) {
        const double b = pick(mix(seed ^ (2 * i)), mode);
        const double a0 = pick(mix(seed ^ (2 * i + 1)), mode);
        const double a1 = pick(mix(seed ^ (2 * i + 1) ^ 0x5555), mode);
        out[2 * i] = a0 / b;
        out[2 * i + 1] = a1 / b;
    }
}
__global__ void k_cmp(uint64_t n, const double* x, const double* y, const unsigned char* fast,
                      unsigned long long* bad, unsigned long long* slow) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x) {
        if (!fast[i]) {
            atomicAdd(slow, 1ull);
            continue;
        }
        if (__double_as_longlong(x[2 * i]) != __double_as_longlong(y[2 * i]) ||
            __double_as_longlong(x[2 * i + 1]) != __double_as_longlong(y[2 * i + 1]))
            atomicAdd(bad, 1ull);
    }
}

int main() {
    unsigned long long *d, h[2];
    cudaMalloc(&d, 16);
    int fail = 0;
    for (int mode = 0; mode < 2; ++mode) {
        cudaMemset(d, 0, 16);
        const uint64_t n = 1ull << 28;
        double *x, *y;
        unsigned char* f;
        cudaMalloc(&x, n * 16);
        cudaMalloc(&y, n * 16);
        cudaMalloc(&f, n);
        for (int rep = 0; rep < 4; ++rep) {
            const uint64_t seed = 0x1510035601ull + 7919ull * (mode * 4 + rep);
            k_mine<<<148 * 16, 256>>>(n, seed, mode, x, f);
            k_stock<<<148 * 16, 256>>>(n, seed, mode, y);
            k_cmp<<<148 * 16, 256>>>(n, x, y, f, d, d + 1);
        }
        cudaFree(x);
        cudaFree(y);
        cudaFree(f);
        cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
        printf("mode %d: %llu pairs x 2 quotients, mismatches %llu, slow-path groups %llu\n", mode,
               (unsigned long long)(4 * n), h[0], h[1]);
        fail |= h[0] != 0;
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        printf("cuda error %s\n", cudaGetErrorString(e));
        return 2;
    }
    return fail;
}
