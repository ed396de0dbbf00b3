// Microbenchmark: shared-memory wavefront cost of the lookup / gather patterns considered for the EM kernel.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o lds_patterns lds_patterns.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int kIters = 4096;
constexpr int kUnroll = 8;

template <int MODE>
__global__ void __launch_bounds__(512, 1) bench(const uint32_t* __restrict__ idx, float* out, long long* cycles) {
    extern __shared__ __align__(16) unsigned char sm[];
    float* fs = reinterpret_cast<float*>(sm);
    for (int i = threadIdx.x; i < 16384; i += blockDim.x) fs[i] = 1.0f + (i & 7);
    __syncthreads();
    // per-thread index stream (8 values, reused): random nibbles / random slots
    uint32_t ix[kUnroll];
    for (int u = 0; u < kUnroll; ++u) ix[u] = idx[(blockIdx.x * blockDim.x + threadIdx.x) * kUnroll + u];
    float a0 = 0, a1 = 0, a2 = 0, a3 = 0;
    const int lane = threadIdx.x & 31;
    __syncthreads();
    const long long t0 = clock64();
    for (int it = 0; it < kIters; ++it) {
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            uint32_t r = ix[u];
            if (MODE == 0) {  // LDS.32, 16-entry table (64 B)
                a0 += fs[u * 16 + (r & 15)];
            } else if (MODE == 1) {  // LDS.64, 16 entries x 8 B
                const float2 v = reinterpret_cast<const float2*>(fs)[u * 16 + (r & 15)];
                a0 += v.x; a1 += v.y;
            } else if (MODE == 2) {  // LDS.128, 16 entries x 16 B
                const float4 v = reinterpret_cast<const float4*>(fs)[u * 16 + (r & 15)];
                a0 += v.x; a1 += v.y; a2 += v.z; a3 += v.w;
            } else if (MODE == 3) {  // LDS.32, 64-entry table
                a0 += fs[u * 64 + (r & 63)];
            } else if (MODE == 4) {  // LDS.32 gather, distinct mod 32
                a0 += fs[((r >> 8) & 0xFE0) + ((lane + u) & 31)];
            } else if (MODE == 5) {  // LDS.64 gather: slot distinct mod 16 within each half-warp
                const float2 v = reinterpret_cast<const float2*>(fs)[((r >> 8) & 0xFF0) + ((lane + u) & 15)];
                a0 += v.x; a1 += v.y;
            } else if (MODE == 6) {  // LDS.128 gather: slot distinct mod 8 within each quarter-warp
                const float4 v = reinterpret_cast<const float4*>(fs)[((r >> 8) & 0x7F8) + ((lane + u) & 7)];
                a0 += v.x; a1 += v.y; a2 += v.z; a3 += v.w;
            } else if (MODE == 7) {  // LDS.64 gather: slot distinct mod 32 over the whole warp (only)
                const float2 v = reinterpret_cast<const float2*>(fs)[((r >> 8) & 0x7E0) + ((lane * 5 + u) & 31)];
                a0 += v.x; a1 += v.y;
            } else if (MODE == 8) {  // LDS.128 16-entry where entries e and e+8 never both appear in a quarter (r&7 only)
                const float4 v = reinterpret_cast<const float4*>(fs)[u * 16 + (r & 7) + ((lane >> 3) & 1) * 8];
                a0 += v.x; a1 += v.y; a2 += v.z; a3 += v.w;
            } else if (MODE == 9) {  // LDS.64 256-entry x 8 B random (4-column tables, 2 buckets)
                const float2 v = reinterpret_cast<const float2*>(fs)[u * 256 + (r & 255)];
                a0 += v.x; a1 += v.y;
            } else if (MODE == 10) {  // LDS.32 256-entry random
                a0 += fs[u * 256 + (r & 255)];
            } else if (MODE == 11) {  // LDS.64, 64 entries x 8 B random (3-column tables, 2 buckets)
                const float2 v = reinterpret_cast<const float2*>(fs)[u * 64 + (r & 63)];
                a0 += v.x; a1 += v.y;
            }
            ix[u] = r;
        }
        // rotate so the compiler cannot hoist (cheap ALU)
        uint32_t t = ix[0];
#pragma unroll
        for (int u = 0; u + 1 < kUnroll; ++u) ix[u] = ix[u + 1];
        ix[kUnroll - 1] = t;
    }
    const long long t1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3;
    if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

template <int MODE>
void run(const char* name, const uint32_t* idx, float* out, long long* cyc, int warps) {
    cudaFuncSetAttribute(bench<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
    bench<MODE><<<148, warps * 32, 65536>>>(idx, out, cyc);
    cudaDeviceSynchronize();
    bench<MODE><<<148, warps * 32, 65536>>>(idx, out, cyc);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[148];
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    double avg = 0;
    for (int i = 0; i < 148; ++i) avg += h[i];
    avg /= 148;
    const double n_inst = double(kIters) * kUnroll * warps;
    printf("%-58s warps=%2d  %.3f cyc per warp-LDS per SM  (%s)\n", name, warps, avg / n_inst, cudaGetErrorString(e));
}

int main() {
    const int n = 148 * 512 * kUnroll;
    uint32_t* h = new uint32_t[n];
    uint64_t s = 88172645463325252ULL;
    for (int i = 0; i < n; ++i) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; h[i] = uint32_t(s >> 16); }
    uint32_t* d; float* out; long long* cyc;
    cudaMalloc(&d, n * 4); cudaMalloc(&out, 148 * 512 * 4); cudaMalloc(&cyc, 148 * 8);
    cudaMemcpy(d, h, n * 4, cudaMemcpyHostToDevice);
    for (int warps : {8, 16}) {
        run<0>("LDS.32  16-entry table (pair, 1 bucket)", d, out, cyc, warps);
        run<1>("LDS.64  16-entry x 8B (pair, 2 buckets)", d, out, cyc, warps);
        run<2>("LDS.128 16-entry x 16B (pair, 4 buckets)", d, out, cyc, warps);
        run<8>("LDS.128 16-entry x 16B, no e/e+8 clash inside a quarter", d, out, cyc, warps);
        run<3>("LDS.32  64-entry table (triple, 1 bucket)", d, out, cyc, warps);
        run<11>("LDS.64  64-entry x 8B (triple, 2 buckets)", d, out, cyc, warps);
        run<10>("LDS.32  256-entry table (quad, 1 bucket)", d, out, cyc, warps);
        run<9>("LDS.64  256-entry x 8B (quad, 2 buckets)", d, out, cyc, warps);
        run<4>("LDS.32  gather distinct mod 32", d, out, cyc, warps);
        run<5>("LDS.64  gather distinct mod 16 per half", d, out, cyc, warps);
        run<7>("LDS.64  gather distinct mod 32 whole warp only", d, out, cyc, warps);
        run<6>("LDS.128 gather distinct mod 8 per quarter", d, out, cyc, warps);
    }
    return 0;
}
