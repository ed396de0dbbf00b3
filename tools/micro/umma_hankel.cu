// Probe: can the EM sweeps be fed to the 5th-generation tensor cores without ever materialising the one-hot
// window matrix?  For a sequence s the E-step weights of 128 buckets are  S[b][j] = sum_c D_b[c][s_{j+c}]
// = D[128 x 4l] * H[4l x W]  with H[(c,r)][j] = [s_{j+c} == r], and the M-step counts are O = P[128 x W] * H^T.
// H is a Hankel matrix: row (c,r) of window j is the one-hot of base position j + c.  Stored as a flat array of
// 8-byte one-hot codes (4 x bf16 per base), window j's 4l entries are the 8l bytes starting at byte 8j — so the
// canonical NO-SWIZZLE shared-memory layouts of tcgen05.mma describe H directly, with overlapping core matrices:
//   * K-major B of GEMM1 (N = windows, K = (c,r)): rows 16 B apart => rows are the EVEN windows of a copy that
//     starts at an even base (the ODD windows use a second copy shifted by one base); LBO = 16 B, SBO = 128 B;
//   * MN-major B of GEMM2 (N = (c,r), K = windows): SBO = 16 B, LBO = 128 B.
// This program checks both against a CPU computation (SS and TS operand modes) and times the instruction
// streams.  Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o umma_hankel umma_hankel.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>
#include <cuda_bf16.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); exit(2); } } while (0)

constexpr int kM = 128;      // buckets per tile
constexpr int kKc = 16;      // columns (base positions per window) covered: K = 4 * kKc = 64
constexpr int kK = 4 * kKc;
constexpr int kNmax = 256;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
    uint64_t d = 0;
    d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFF);
    d |= static_cast<uint64_t>((lbo_bytes >> 4) & 0x3FFF) << 16;
    d |= static_cast<uint64_t>((sbo_bytes >> 4) & 0x3FFF) << 32;
    d |= 1ULL << 46;  // descriptor version (Blackwell)
    return d;         // base offset 0, absolute LBO mode, SWIZZLE_NONE
}

// kind::f16, A/B bf16, FP32 accumulate, M = 128
__host__ __device__ constexpr uint32_t make_idesc(int n, bool b_mn_major) {
    return (1u << 4) | (1u << 7) | (1u << 10) | ((b_mn_major ? 1u : 0u) << 16) | (static_cast<uint32_t>(n >> 3) << 17) |
           (static_cast<uint32_t>(kM >> 4) << 24);
}

__device__ __forceinline__ void mma_ss(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc, bool acc) {
    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n"
                 :: "r"(d_tmem), "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc ? 1u : 0u) : "memory");
}
__device__ __forceinline__ void mma_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc, bool acc) {
    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n"
                 :: "r"(d_tmem), "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(acc ? 1u : 0u) : "memory");
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, int count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile("{\n.reg .pred P1;\nWAIT_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@P1 bra DONE_%=;\nbra WAIT_%=;\nDONE_%=:\n}\n"
                 :: "r"(smem_u32(bar)), "r"(parity) : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]),
                   "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),
                   "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]),
                   "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
                 : "r"(taddr));
}
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};"
                 :: "r"(taddr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
                    "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]),
                    "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]),
                    "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31]) : "memory");
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

struct Params {
    const uint8_t* seq;        // 2-bit symbols, one per byte, length n_bases
    int n_bases;
    int n_win_half;            // N of GEMM1 per parity (even windows / odd windows), multiple of 16, <= 256
    const __nv_bfloat16* A;    // [kM][kK] row-major log-odds (one bf16 term)
    const __nv_bfloat16* P;    // [kM][2 * n_win_half]: responsibilities, column i = even window 2i for i < n_win_half, then odd windows
    float* S_ss;               // [2][kM][n_win_half]  GEMM1, A from shared memory
    float* S_ts;               // [2][kM][n_win_half]  GEMM1, A from tensor memory
    float* O_ts;               // [kM][kK]             GEMM2, A (= P) from tensor memory, B MN-major
    long long* cycles;         // [8] timings
    int reps;
    int swap2;                 // 1: exchange LBO and SBO of the MN-major descriptor (semantics check)
};

// shared memory: E0 | E1 | A tile (canonical K-major, no swizzle) | barriers
__global__ void __launch_bounds__(128, 1) probe(const Params p) {
    extern __shared__ __align__(128) unsigned char smem[];
    const int e_bytes = ((p.n_bases + 2) * 8 + 127) & ~127;
    unsigned char* E0 = smem;                 // base position q at byte 8q
    unsigned char* E1 = smem + e_bytes;       // base position q+1 at byte 8q
    unsigned char* As = smem + 2 * e_bytes;   // [kK/8 chunks][kM rows][8 bf16]
    uint64_t* bar = reinterpret_cast<uint64_t*>(As + kM * kK * 2);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 2);
    const int tid = threadIdx.x, warp = tid >> 5;

    // ---- operands into shared memory
    for (int q = tid; q < p.n_bases + 2; q += blockDim.x) {
        uint64_t code0 = 0, code1 = 0;
        if (q < p.n_bases) code0 = 0x3F80ULL << (16 * p.seq[q]);           // bf16 1.0 at slot r
        if (q + 1 < p.n_bases) code1 = 0x3F80ULL << (16 * p.seq[q + 1]);
        *reinterpret_cast<uint64_t*>(E0 + 8 * q) = code0;
        *reinterpret_cast<uint64_t*>(E1 + 8 * q) = code1;
    }
    for (int e = tid; e < kM * kK; e += blockDim.x) {
        const int row = e / kK, kk = e % kK;
        reinterpret_cast<__nv_bfloat16*>(As)[(kk / 8) * (kM * 8) + row * 8 + (kk % 8)] = p.A[e];
    }
    if (tid == 0) {
        mbar_init(&bar[0], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    fence_async_smem();
    __syncthreads();
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" :: "r"(smem_u32(tmem_slot)), "r"(512u) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tmem = *tmem_slot;
    const uint32_t lane_base = static_cast<uint32_t>(warp * 32) << 16;
    const int N = p.n_win_half;
    uint32_t phase = 0;
    // TMEM map: [0, 256) S accumulator; [256, 288) A (64 bf16 = 32 columns); [288, 288 + N) P (2N bf16); [448, 512) O
    const uint32_t tS = tmem, tA = tmem + 256, tP = tmem + 288, tO = tmem + 448;

    // ---- A and P into tensor memory (thread = row)
    {
        uint32_t r[32];
        const uint32_t* arow = reinterpret_cast<const uint32_t*>(p.A + static_cast<size_t>(tid) * kK);
        for (int i = 0; i < 32; ++i) r[i] = arow[i];
        tmem_st32(tA + lane_base, r);
        const uint32_t* prow = reinterpret_cast<const uint32_t*>(p.P + static_cast<size_t>(tid) * 2 * N);
        for (int c0 = 0; c0 < N; c0 += 32) {  // N columns of packed pairs (2N bf16); N is a multiple of 16: pad reads with 0
            for (int i = 0; i < 32; ++i) r[i] = c0 + i < N ? prow[c0 + i] : 0u;
            if (c0 + 32 <= 160) tmem_st32(tP + lane_base + c0, r);
        }
        tmem_wait_st();
    }
    fence_before();
    __syncthreads();
    fence_after();

    const uint32_t idesc1 = make_idesc(N, false);
    const uint32_t idesc2 = make_idesc(kK, true);
    for (int mode = 0; mode < 2; ++mode) {        // 0: A from shared memory, 1: A from tensor memory
        for (int par = 0; par < 2; ++par) {       // even / odd windows
            const unsigned char* E = par ? E1 : E0;
            if (tid == 0) {
                for (int kb = 0; kb < kK / 16; ++kb) {
                    const uint64_t bdesc = make_desc(smem_u32(E) + 32 * kb, 16, 128);
                    if (mode == 0) {
                        const uint64_t adesc = make_desc(smem_u32(As) + kb * 2 * (kM * 16), kM * 16, 128);
                        mma_ss(tS, adesc, bdesc, idesc1, kb > 0);
                    } else {
                        mma_ts(tS, tA + 8 * kb, bdesc, idesc1, kb > 0);
                    }
                }
                mma_commit(&bar[0]);
            }
            mbar_wait(&bar[0], phase);
            phase ^= 1;
            fence_after();
            float* out = (mode ? p.S_ts : p.S_ss) + (static_cast<size_t>(par) * kM + tid) * N;
            for (int c0 = 0; c0 < N; c0 += 32) {
                uint32_t r[32];
                tmem_ld32(tS + lane_base + c0, r);
                tmem_wait_ld();
                for (int i = 0; i < 32 && c0 + i < N; ++i) out[c0 + i] = __uint_as_float(r[i]);
            }
            fence_before();
            __syncthreads();
            fence_after();
        }
    }
    // ---- GEMM2: O[128 x 64] = sum over even windows i: P[b][i] * onehot(base 2i + c), then odd windows
    if (tid == 0) {
        bool acc = false;
        for (int par = 0; par < 2; ++par) {
            const unsigned char* E = par ? E1 : E0;
            for (int kb = 0; kb < N / 16; ++kb) {
                const uint64_t bdesc = p.swap2 ? make_desc(smem_u32(E) + 16 * 16 * kb, 16, 128) : make_desc(smem_u32(E) + 16 * 16 * kb, 128, 16);
                mma_ts(tO, tP + (par * N + 16 * kb) / 2, bdesc, idesc2, acc);
                acc = true;
            }
        }
        mma_commit(&bar[0]);
    }
    mbar_wait(&bar[0], phase);
    phase ^= 1;
    fence_after();
    for (int c0 = 0; c0 < kK; c0 += 32) {
        uint32_t r[32];
        tmem_ld32(tO + lane_base + c0, r);
        tmem_wait_ld();
        for (int i = 0; i < 32; ++i) p.O_ts[static_cast<size_t>(tid) * kK + c0 + i] = __uint_as_float(r[i]);
    }
    fence_before();
    __syncthreads();
    fence_after();

    // ---- timings (one CTA alone on its SM)
    // [0] GEMM1 TS: reps x (4 MMAs, N columns)   [1] GEMM1 SS   [2] GEMM2 TS: reps x (N/16 MMAs, 64 columns)
    for (int which = 0; which < 3; ++which) {
        __syncthreads();
        const long long t0 = clock64();
        if (tid == 0) {
            for (int rep = 0; rep < p.reps; ++rep) {
                if (which < 2) {
                    for (int kb = 0; kb < kK / 16; ++kb) {
                        const uint64_t bdesc = make_desc(smem_u32(E0) + 32 * kb, 16, 128);
                        if (which == 1) {
                            const uint64_t adesc = make_desc(smem_u32(As) + kb * 2 * (kM * 16), kM * 16, 128);
                            mma_ss(tS, adesc, bdesc, idesc1, true);
                        } else {
                            mma_ts(tS, tA + 8 * kb, bdesc, idesc1, true);
                        }
                    }
                } else {
                    for (int kb = 0; kb < N / 16; ++kb) {
                        const uint64_t bdesc = make_desc(smem_u32(E0) + 16 * 16 * kb, 128, 16);
                        mma_ts(tO, tP + (16 * kb) / 2, bdesc, idesc2, true);
                    }
                }
            }
            mma_commit(&bar[0]);
        }
        mbar_wait(&bar[0], phase);
        phase ^= 1;
        fence_after();
        const long long t1 = clock64();
        if (tid == 0) p.cycles[which] = t1 - t0;
    }
    // [3] tensor-memory read: every warp reads its 32 lanes x N columns, reps times
    {
        __syncthreads();
        const long long t0 = clock64();
        uint32_t accv = 0;
        for (int rep = 0; rep < p.reps; ++rep) {
            for (int c0 = 0; c0 + 32 <= N; c0 += 32) {
                uint32_t r[32];
                tmem_ld32(tS + lane_base + c0, r);
                tmem_wait_ld();
                for (int i = 0; i < 32; ++i) accv ^= r[i];
            }
        }
        __syncthreads();
        const long long t1 = clock64();
        if (tid == 0) p.cycles[3] = t1 - t0;
        if (accv == 0x12345678u) p.cycles[7] = 1;
    }
    // [4] softmax-style pass over the S tile: ld, ex2, sum, split into bf16 hi/lo, store as P, reps times
    {
        __syncthreads();
        const long long t0 = clock64();
        float sum = 0.f, mx = -1e30f;
        for (int rep = 0; rep < p.reps; ++rep) {
            for (int c0 = 0; c0 + 32 <= N && c0 + 32 <= 160; c0 += 32) {
                uint32_t r[32], o[32];
                tmem_ld32(tS + lane_base + c0, r);
                tmem_wait_ld();
#pragma unroll
                for (int i = 0; i < 32; i += 2) {
                    const float w0 = __uint_as_float(r[i]), w1 = __uint_as_float(r[i + 1]);
                    mx = fmaxf(mx, fmaxf(w0, w1));
                    float e0, e1;
                    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e0) : "f"(w0 * 1.442695f - 30.f));
                    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e1) : "f"(w1 * 1.442695f - 30.f));
                    sum += e0 + e1;
                    const __nv_bfloat162 hi = __floats2bfloat162_rn(e0, e1);
                    const float2 hf = __bfloat1622float2(hi);
                    const __nv_bfloat162 lo = __floats2bfloat162_rn(e0 - hf.x, e1 - hf.y);
                    o[i / 2] = *reinterpret_cast<const uint32_t*>(&hi);
                    o[16 + i / 2] = *reinterpret_cast<const uint32_t*>(&lo);
                }
                tmem_st32(tP + lane_base + c0, o);
            }
            tmem_wait_st();
        }
        __syncthreads();
        const long long t1 = clock64();
        if (tid == 0) p.cycles[4] = t1 - t0;
        if (sum + mx == 0.12345f) p.cycles[7] = 2;
    }
    fence_before();
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(tmem), "r"(512u) : "memory");
}

static float bf(float v) { return __bfloat162float(__float2bfloat16(v)); }

int main(int argc, char** argv) {
    const int N = argc > 1 ? atoi(argv[1]) : 144;  // windows per parity (multiple of 16, <= 160 here: P fits 160 columns)
    const int reps = argc > 2 ? atoi(argv[2]) : 200;
    if (N % 16 != 0 || N < 16 || N > 160) { printf("N must be a multiple of 16 in [16,160]\n"); return 1; }
    const int n_bases = 2 * N + kKc + 2;
    srand(12345);
    std::vector<uint8_t> seq(n_bases);
    for (auto& v : seq) v = rand() & 3;
    std::vector<__nv_bfloat16> A(kM * kK), P(kM * 2 * N);
    std::vector<float> Af(kM * kK), Pf(kM * 2 * N);
    for (int i = 0; i < kM * kK; ++i) { Af[i] = bf(-20.f * (rand() / float(RAND_MAX)) + 1.f); A[i] = __float2bfloat16(Af[i]); }
    for (int i = 0; i < kM * 2 * N; ++i) { Pf[i] = bf(rand() / float(RAND_MAX)); P[i] = __float2bfloat16(Pf[i]); }

    uint8_t* d_seq; __nv_bfloat16 *d_A, *d_P; float *d_Sss, *d_Sts, *d_O; long long* d_cyc;
    CK(cudaMalloc(&d_seq, n_bases)); CK(cudaMalloc(&d_A, A.size() * 2)); CK(cudaMalloc(&d_P, P.size() * 2));
    CK(cudaMalloc(&d_Sss, sizeof(float) * 2 * kM * N)); CK(cudaMalloc(&d_Sts, sizeof(float) * 2 * kM * N));
    CK(cudaMalloc(&d_O, sizeof(float) * kM * kK)); CK(cudaMalloc(&d_cyc, 64));
    CK(cudaMemcpy(d_seq, seq.data(), n_bases, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_A, A.data(), A.size() * 2, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_P, P.data(), P.size() * 2, cudaMemcpyHostToDevice));
    CK(cudaMemset(d_Sss, 0xFF, sizeof(float) * 2 * kM * N)); CK(cudaMemset(d_Sts, 0xFF, sizeof(float) * 2 * kM * N));
    CK(cudaMemset(d_O, 0xFF, sizeof(float) * kM * kK)); CK(cudaMemset(d_cyc, 0, 64));
    Params p{d_seq, n_bases, N, d_A, d_P, d_Sss, d_Sts, d_O, d_cyc, reps, argc > 3 ? atoi(argv[3]) : 0};
    const int e_bytes = ((n_bases + 2) * 8 + 127) & ~127;
    const size_t smem = 2 * e_bytes + kM * kK * 2 + 64;
    CK(cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    probe<<<1, 128, smem>>>(p);
    CK(cudaDeviceSynchronize());

    std::vector<float> Sss(2 * kM * N), Sts(2 * kM * N), O(kM * kK);
    long long cyc[8];
    CK(cudaMemcpy(Sss.data(), d_Sss, Sss.size() * 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(Sts.data(), d_Sts, Sts.size() * 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(O.data(), d_O, O.size() * 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(cyc, d_cyc, 64, cudaMemcpyDeviceToHost));

    double err_ss = 0, err_ts = 0, err_o = 0;
    for (int par = 0; par < 2; ++par)
        for (int b = 0; b < kM; ++b)
            for (int i = 0; i < N; ++i) {
                const int j = 2 * i + par;
                double ref = 0;
                for (int c = 0; c < kKc; ++c) ref += Af[b * kK + 4 * c + seq[j + c]];
                err_ss = fmax(err_ss, fabs(ref - Sss[(par * kM + b) * N + i]));
                err_ts = fmax(err_ts, fabs(ref - Sts[(par * kM + b) * N + i]));
            }
    for (int b = 0; b < kM; ++b)
        for (int cr = 0; cr < kK; ++cr) {
            double ref = 0;
            for (int par = 0; par < 2; ++par)
                for (int i = 0; i < N; ++i) {
                    const int j = 2 * i + par;
                    if (seq[j + cr / 4] == cr % 4) ref += Pf[b * 2 * N + par * N + i];
                }
            err_o = fmax(err_o, fabs(ref - O[b * kK + cr]));
        }
    printf("N=%d  GEMM1 (K-major Hankel B, LBO=16 SBO=128): max|err| SS %.3g  TS %.3g   [%s]\n", N, err_ss, err_ts,
           (err_ss < 1e-3 && err_ts < 1e-3) ? "PASS" : "FAIL");
    printf("      GEMM2 (MN-major Hankel B, SBO=16 LBO=128, A = P in TMEM): max|err| %.3g   [%s]\n", err_o, err_o < 1e-3 ? "PASS" : "FAIL");
    printf("      S[0][0..3] ss %.4f %.4f %.4f %.4f   O[0][0..3] %.4f %.4f %.4f %.4f\n", Sss[0], Sss[1], Sss[2], Sss[3], O[0], O[1], O[2], O[3]);
    const double mma1 = 4.0 * reps, mma2 = (N / 16.0) * reps;
    printf("timing (1 CTA): GEMM1 TS %.1f cyc/MMA (floor %.1f)  GEMM1 SS %.1f cyc/MMA  GEMM2 TS %.1f cyc/MMA (floor %.1f)\n",
           cyc[0] / mma1, 128.0 * N / 256.0, cyc[1] / mma1, cyc[2] / mma2, 128.0 * 64 / 256.0);
    const int cols = (N / 32) * 32, cols4 = cols < 160 ? cols : 160;
    printf("        TMEM ld: %.2f cyc per 32x32 block per warp (4 warps) => %.1f B/clk/SM\n", double(cyc[3]) / (reps * (cols / 32)),
           4.0 * 32 * 32 * 4 * reps * (cols / 32) / double(cyc[3]));
    printf("        softmax-style pass (ld, ex2, sum, max, bf16 hi/lo split, TMEM st): %.2f cyc per element-row-of-32 => %.2f elements/clk/SM with 4 warps\n",
           double(cyc[4]) / (reps * (cols4 / 32) * 32.0), 128.0 * reps * cols4 / double(cyc[4]));
    return (err_ss < 1e-3 && err_ts < 1e-3 && err_o < 1e-3) ? 0 : 1;
}
