// Microbenchmark: do warp shuffles share throughput with shared-memory loads?  (cycles per loop trip on one SM)
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o shfl_vs_lds shfl_vs_lds.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int kIters = 4096;

template <int N_LDS, int N_SHFL>
__global__ void __launch_bounds__(512, 1) bench(const uint32_t* __restrict__ idx, float* out, long long* cycles) {
    __shared__ float2 tab[8][16];
    for (int i = threadIdx.x; i < 128; i += blockDim.x) tab[i / 16][i % 16] = make_float2(1.f + i, 2.f + i);
    __syncthreads();
    uint32_t r = idx[blockIdx.x * blockDim.x + threadIdx.x];
    float regs[8];
    for (int k = 0; k < 8; ++k) regs[k] = 1.f + k + (threadIdx.x & 15);
    float a0 = 0, a1 = 0;
    __syncthreads();
    const long long t0 = clock64();
    for (int it = 0; it < kIters; ++it) {
#pragma unroll
        for (int k = 0; k < N_LDS; ++k) {
            const float2 v = tab[k][(r >> (4 * k)) & 15];
            a0 += v.x;
            a1 += v.y;
        }
#pragma unroll
        for (int k = 0; k < N_SHFL; ++k) {
            a0 += __shfl_sync(0xffffffffu, regs[k & 7], (r >> (4 * (k & 7))) & 15);
        }
        r = r * 1664525u + 1013904223u;
    }
    const long long t1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1;
    if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

template <int N_LDS, int N_SHFL>
void run(const uint32_t* idx, float* out, long long* cyc, int warps) {
    bench<N_LDS, N_SHFL><<<148, warps * 32>>>(idx, out, cyc);
    cudaDeviceSynchronize();
    bench<N_LDS, N_SHFL><<<148, warps * 32>>>(idx, out, cyc);
    cudaDeviceSynchronize();
    long long h[148];
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    double avg = 0;
    for (int i = 0; i < 148; ++i) avg += h[i];
    avg /= 148;
    printf("LDS.64 x%d + SHFL x%-2d  warps=%2d  %.2f cycles per trip per warp (SM-wide: %.2f per warp-trip)\n", N_LDS, N_SHFL, warps,
           avg / kIters, avg / kIters / warps);
}

int main() {
    const int n = 148 * 512;
    uint32_t* h = new uint32_t[n];
    uint64_t s = 88172645463325252ULL;
    for (int i = 0; i < n; ++i) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; h[i] = uint32_t(s >> 16); }
    uint32_t* d; float* out; long long* cyc;
    cudaMalloc(&d, n * 4); cudaMalloc(&out, n * 4); cudaMalloc(&cyc, 148 * 8);
    cudaMemcpy(d, h, n * 4, cudaMemcpyHostToDevice);
    for (int warps : {16}) {
        run<8, 0>(d, out, cyc, warps);
        run<0, 8>(d, out, cyc, warps);
        run<0, 16>(d, out, cyc, warps);
        run<4, 8>(d, out, cyc, warps);
        run<8, 8>(d, out, cyc, warps);
        run<4, 0>(d, out, cyc, warps);
    }
    return 0;
}
