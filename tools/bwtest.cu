// bwtest.cu — HBM bandwidth of the fused kernel's access pattern (measurement
// tool, not product code).  Block pool [tile][comp][dir][z][y][x] FP64, E = 32.
//   mode 0: flat copy of the whole pool (grid-stride, 16 B per thread)
//   mode 1: k_main pattern — CTA = 32 x BY column block of one tile, marching
//           z; per plane each thread reads its cell's 19*C values (x-shifted
//           pull for ex != 0) and writes 19*C values; all loads in flight
//   mode 2: as 1 with unshifted reads (aligned rows)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o bwtest tools/bwtest.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

constexpr int E = 32, E3 = E * E * E, Q = 19;
__constant__ int EX[Q] = {0, 1, -1, 0, 0, 0, 0, 1, -1, 1, -1, 1, -1, 1, -1, 0, 0, 0, 0};

template <int C, int BY, bool SHIFT>
__global__ void __launch_bounds__(32 * BY) k_pattern(const double* __restrict__ src, double* __restrict__ dst) {
    const int tile = blockIdx.x / (E / BY);
    const int y = (blockIdx.x % (E / BY)) * BY + threadIdx.x / 32;
    const int x = threadIdx.x % 32;
    const double* s = src + size_t(tile) * C * Q * E3;
    double* d = dst + size_t(tile) * C * Q * E3;
    for (int z = 0; z < E; ++z) {
        const int cell = (z * E + y) * E + x;
        double v[C * Q];
#pragma unroll
        for (int k = 0; k < C * Q; ++k) {
            int xs = x;
            if (SHIFT) xs = (x - EX[k % Q]) & (E - 1);
            v[k] = __ldg(s + size_t(k) * E3 + (z * E + y) * E + xs);
        }
#pragma unroll
        for (int k = 0; k < C * Q; ++k) d[size_t(k) * E3 + cell] = v[k] + 1.0;
    }
}

__global__ void k_copy(const double2* __restrict__ s, double2* __restrict__ d, size_t n) {
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x)
        d[i] = s[i];
}

int main(int argc, char** argv) {
    const int tiles = argc > 1 ? atoi(argv[1]) : 504;
    constexpr int C = 2;
    const size_t n = size_t(tiles) * C * Q * E3;
    double *a, *b;
    cudaMalloc(&a, n * 8);
    cudaMalloc(&b, n * 8);
    cudaMemset(a, 0, n * 8);
    cudaMemset(b, 0, n * 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto run = [&](const char* name, auto launch) {
        for (int w = 0; w < 3; ++w) launch();
        cudaEventRecord(e0);
        const int reps = 10;
        for (int r = 0; r < reps; ++r) launch();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        ms /= reps;
        printf("%-34s %8.3f ms  %8.1f GB/s (read+write)\n", name, ms, 2.0 * n * 8 / (ms * 1e-3) / 1e9);
    };
    run("flat copy", [&] { k_copy<<<148 * 8, 512>>>((double2*)a, (double2*)b, n / 2); });
    run("pattern BY=8 shifted", [&] { k_pattern<C, 8, true><<<tiles * 4, 256>>>(a, b); });
    run("pattern BY=8 aligned", [&] { k_pattern<C, 8, false><<<tiles * 4, 256>>>(a, b); });
    run("pattern BY=4 shifted", [&] { k_pattern<C, 4, true><<<tiles * 8, 128>>>(a, b); });
    run("pattern BY=16 shifted", [&] { k_pattern<C, 16, true><<<tiles * 2, 512>>>(a, b); });
    run("pattern BY=32 shifted", [&] { k_pattern<C, 32, true><<<tiles, 1024>>>(a, b); });
    cudaError_t err = cudaGetLastError();
    if (err != cudaSuccess) printf("error %s\n", cudaGetErrorString(err));
    return 0;
}
