// pm_em_tc.cuh — EM refinement on the 5th-generation tensor cores: 128 enriched buckets per CTA in lockstep.
//
// Per bucket the E-step is a table walk, but across the buckets of a batch it IS a contraction over a matrix that
// every bucket shares.  For one sequence s with W windows (refine.hpp:150-203, :227-237):
//     E-step   S[b][j]   = sum_c D_b[c][s_{j+c}]                  = D[128 x 4l] * H[4l x W]
//     M-step   O[b][c,r] = sum_j e[b][j] * [s_{j+c} == r]         = P[128 x W] * H^T[W x 4l]
// with D_b the log-odds table of bucket b, H[(c,r)][j] = [s_{j+c} == r] the one-hot window matrix and
// e = exp(S - ref) the un-normalised responsibilities (normalised per sequence after the fact).  H is never
// materialised: it is a Hankel matrix, so with the sequence stored as a flat array of 8-byte one-hot codes
// (4 x bf16 per base) window j's 4l entries are the 8l bytes that start at byte 8j, and the canonical NO-SWIZZLE
// shared-memory operand layouts of tcgen05.mma describe it with OVERLAPPING core matrices:
//     GEMM1  B K-major   (N = windows, K = (c,r)):  rows are 16 B apart => the even windows of an array that starts
//                         at base 0, the odd windows of a copy shifted by one base;  LBO = 16 B, SBO = 128 B
//     GEMM2  B MN-major  (N = (c,r), K = windows):  SBO = 16 B, LBO = 128 B
// (tools/micro/umma_hankel.cu checks both descriptors against a CPU computation).  A operands live in tensor
// memory: D as three bf16 terms (hi + mid + lo = 24 significant bits, what FP32 holds), P as two bf16 terms
// written IN PLACE over the S block it was computed from; accumulation is FP32 in tensor memory.
//
// Roles (384 threads): warps 0-7 = two warpgroups of "softmax" threads, thread = bucket row, the warpgroups
// split the columns of every block; warp 8 lane 0 issues every tcgen05.mma; warp 9 expands the next sequence
// into the one-hot arrays.  mbarriers connect them (full/empty pairs), tcgen05.commit signals MMA completion.
//
// What this kernel does NOT do is the FP64 work that makes the discrete outputs reproducible in the saturated
// cases (the near-maximum windows of pm_em_pair.cuh).  Instead it FLAGS a bucket whenever one of its decisions
// is closer than the FP32 error of the tensor-core sums: a likelihood gain that could be below tol
// (refine.hpp:300), an argmax whose runner-up lies within delta, a maximum that left the range of the
// reference.  Flagged buckets are re-run by em_refine_pair_kernel (launch_em in pm_capi.cu) into the same
// output slots; for every other bucket iterations, positions, score and consensus are decided with margin.
#pragma once
#include <cuda_bf16.h>

#include "pm_em_pair.cuh"

namespace pm {
namespace k {

constexpr int kTcRows = 128;        // buckets per CTA tile = MMA M
constexpr int kTcSoftWarps = 8;     // two warpgroups
constexpr int kTcThreads = 384;     // + a third warpgroup: MMA warp, producer warp, two idle warps (it gives its registers away)
constexpr int kTcMaxSeqs = 64;      // previous maxima [t][128] live in shared memory
constexpr int kTcMaxIters = 8;      // no early exit for a tile: larger budgets use the pair kernel
constexpr int kTcMaxL = 20;         // K = 4 * KC <= 80
constexpr int kTcEPad = 96;         // zero one-hot codes behind every sequence (pad windows read them)

enum : unsigned { kTcFlagConv = 1u, kTcFlagRange = 2u, kTcFlagTie = 4u, kTcFlagBad = 8u, kTcFlagSmall = 16u };

// One S/P block of a sweep: up to NBLK columns (a multiple of 32) of ONE sequence.  A column is a window; a
// block consists of one or two MMA segments, each a run of windows of one parity.
struct TcSeg {
    uint16_t par;    // 0: even windows, 1: odd windows
    uint16_t i0;     // first window of the segment, counted within its parity (window j = 2 i + par)
    uint16_t n;      // columns (multiple of 16)
    uint16_t col;    // first column within the block
    uint16_t valid;  // leading columns that are real windows
    uint16_t pad;
};
struct TcBlock {
    uint16_t seq;
    uint16_t ncols;  // multiple of 32; columns beyond the segments are dead
    uint16_t first;  // first block of its sequence
    uint16_t last;   // last block of its sequence
    TcSeg seg[2];    // seg[1].n == 0 when unused
};

struct TcExtra {
    const TcBlock* blocks;  // one sweep = every sequence once, in order
    int n_blocks;
    int e_positions;        // one-hot codes per array (longest sequence + kTcEPad, multiple of 16)
    unsigned char* out_flag;  // [work] kTcFlag* bits; nonzero => the work item must be redone by the exact kernel
    float tie_delta;        // argmax runner-up margin (natural-log units)
    float ll_margin;        // likelihood gains below tol + margin are not decided here
    unsigned long long* stats;  // [4] flagged counts by kind (conv, range, tie, bad)
    unsigned int min_work;      // fewer work items than this: hand every bucket to the pair kernel (a tile's ~1 ms of
                                // sequential passes is a latency floor that a few hundred buckets do not amortise)
};

// ---------------------------------------------------------------------------------------------------------
// PTX wrappers
// ---------------------------------------------------------------------------------------------------------
__device__ __forceinline__ void tc_mbar_arrive(unsigned long long* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void tc_wait(unsigned long long* bar, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "TC_WAIT:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@p bra TC_DONE;\n"
        "bra TC_WAIT;\n"
        "TC_DONE:\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// one lane of a converged warp (the compiler keeps the operands of the guarded instructions in uniform registers)
__device__ __forceinline__ bool tc_elect() {
    uint32_t pred;
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "elect.sync _|p, 0xffffffff;\n"
        "selp.b32 %0, 1, 0, p;\n"
        "}\n"
        : "=r"(pred));
    return pred != 0;
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tc_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tc_commit(unsigned long long* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// D[tmem] (+)= A[tmem] * B[smem descriptor]
__device__ __forceinline__ void tc_mma(uint32_t d_tmem, uint32_t a_tmem, uint32_t b_lo, uint32_t b_hi, uint32_t idesc, bool acc) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        ".reg .b64 bd;\n"
        "setp.ne.b32 p, %5, 0;\n"
        "mov.b64 bd, {%2, %3};\n"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], bd, %4, p;\n"
        "}\n" ::"r"(d_tmem),
        "r"(a_tmem), "r"(b_lo), "r"(b_hi), "r"(idesc), "r"(acc ? 1u : 0u)
        : "memory");
}

// {e1, e0} -> packed bf16x2 (e0 in the low half: the lower K index)
__device__ __forceinline__ uint32_t tc_pack_bf16(float e0, float e1) {
    uint32_t d;
    asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(d) : "f"(e1), "f"(e0));
    return d;
}

__device__ __forceinline__ void tc_ld16(uint32_t taddr, uint32_t* r) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
                   "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                 : "r"(taddr));
}
__device__ __forceinline__ void tc_st16(uint32_t taddr, const uint32_t* r) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
                 "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
                 "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
                 : "memory");
}
__device__ __forceinline__ void tc_ld32(uint32_t taddr, uint32_t (&r)[32]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]),
                   "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),
                   "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]),
                   "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
                 : "r"(taddr));
}
__device__ __forceinline__ void tc_st32(uint32_t taddr, const uint32_t (&r)[32]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
                 "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]), "r"(r[10]),
                 "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]),
                 "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]),
                 "r"(r[31])
                 : "memory");
}

// ---- per-chunk work of a softmax thread: 16 columns (= 16 windows of one parity) of its row ------------------
struct TcSeqState {
    float mxa;            // final pass: running maximum of the weights
    float second;         // final pass: runner-up weight
    int best_j;           // final pass: window of the maximum
};

// EM pass: e = 2^S, as bf16 hi + lo pairs (8 + 8 words) for the M-step GEMM.  S already is weight minus reference
// (the reference is folded into the log-odds terms, see the model update) and the normaliser comes out of GEMM2
// (fold_pending): per pair of columns 2 ex2, 1 byte permute + 2 masks for hi, 1 residual, 1 conversion for lo.
template <bool kMasked>
__device__ __forceinline__ void tc_em_chunk(const uint32_t* __restrict__ r, uint32_t* __restrict__ o, int nvalid) {
#pragma unroll
    for (int k2 = 0; k2 < 16; k2 += 4) {
        float2 w0 = make_float2(__uint_as_float(r[k2]), __uint_as_float(r[k2 + 1]));
        float2 w1 = make_float2(__uint_as_float(r[k2 + 2]), __uint_as_float(r[k2 + 3]));
        if (kMasked) {
            if (k2 >= nvalid) {  // a dead quad (the columns are the same for every row: a uniform branch)
                o[k2 >> 1] = 0u;
                o[(k2 >> 1) + 1] = 0u;
                o[8 + (k2 >> 1)] = 0u;
                o[8 + (k2 >> 1) + 1] = 0u;
                continue;
            }
            if (k2 + 1 >= nvalid) w0.y = -INFINITY;
            if (k2 + 2 >= nvalid) w1.x = -INFINITY;
            if (k2 + 3 >= nvalid) w1.y = -INFINITY;
        }
        const float2 e0 = make_float2(fast_ex2(w0.x), fast_ex2(w0.y));  // 2^-inf = 0 for masked columns
        const float2 e1 = make_float2(fast_ex2(w1.x), fast_ex2(w1.y));
        // hi = the upper 16 bits of e (a byte permute on the ALU pipe: the XU pipe, which the exponentials and the
        // conversions share, is the scarce one), lo = bf16(e - hi): hi + lo carries 15-16 bits of e
        const uint32_t h0 = __byte_perm(__float_as_uint(e0.x), __float_as_uint(e0.y), 0x7632);
        const uint32_t h1 = __byte_perm(__float_as_uint(e1.x), __float_as_uint(e1.y), 0x7632);
        const float2 hf0 = make_float2(__uint_as_float(__float_as_uint(e0.x) & 0xFFFF0000u), __uint_as_float(__float_as_uint(e0.y) & 0xFFFF0000u));
        const float2 hf1 = make_float2(__uint_as_float(__float_as_uint(e1.x) & 0xFFFF0000u), __uint_as_float(__float_as_uint(e1.y) & 0xFFFF0000u));
        const float2 l0 = f2_fma(hf0, make_float2(-1.f, -1.f), e0);  // exact residuals
        const float2 l1 = f2_fma(hf1, make_float2(-1.f, -1.f), e1);
        o[k2 >> 1] = h0;
        o[(k2 >> 1) + 1] = h1;
        o[8 + (k2 >> 1)] = tc_pack_bf16(l0.x, l0.y);
        o[8 + (k2 >> 1) + 1] = tc_pack_bf16(l1.x, l1.y);
    }
}

// final pass: maximum, its window and the runner-up weight, without branches (the rows of a warp are different
// buckets: a data-dependent branch is taken by some lane in nearly every chunk).  The column number within the chunk
// rides in the low four mantissa bits of the weight -- a perturbation below 16 ulp that the tie margin of the caller
// accounts for -- so the running maximum carries its own position; st.best_j is the chunk's first window.
constexpr float kTcFinalUlpMargin = 4e-6f;  // 2 x 15 ulp of a perturbed weight, relative
template <bool kMasked>
__device__ __forceinline__ void tc_final_chunk(const uint32_t* __restrict__ r, int nvalid, int j0, TcSeqState& st) {
    const float m_in = st.mxa;
#pragma unroll
    for (int k2 = 0; k2 < 16; ++k2) {
        float w = __uint_as_float((r[k2] & 0xFFFFFFF0u) | static_cast<uint32_t>(15 - k2));
        if (kMasked && k2 >= nvalid) w = -INFINITY;
        st.second = fmaxf(st.second, fminf(w, st.mxa));
        st.mxa = fmaxf(st.mxa, w);
    }
    st.best_j = st.mxa != m_in ? j0 : st.best_j;
}
__device__ __forceinline__ int tc_final_window(const TcSeqState& st) {
    return st.best_j + 2 * (15 - static_cast<int>(__float_as_uint(st.mxa) & 15u));
}

__device__ __forceinline__ void tc_ld4(uint32_t taddr, uint32_t* r) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];" : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(taddr));
}
__device__ __forceinline__ void tc_st4(uint32_t taddr, const uint32_t* r) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};" ::"r"(taddr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]) : "memory");
}

__device__ __forceinline__ void tc_named_sync() { asm volatile("bar.sync 1, 256;" ::: "memory"); }

// x = hi + mid + lo in bf16 (round to nearest each): 24 significant bits
__device__ __forceinline__ void tc_split3(float x, uint32_t& hi, uint32_t& mid, uint32_t& lo) {
    const __nv_bfloat16 h = __float2bfloat16_rn(x);
    const float r1 = x - __bfloat162float(h);
    const __nv_bfloat16 m = __float2bfloat16_rn(r1);
    const float r2 = r1 - __bfloat162float(m);
    const __nv_bfloat16 l = __float2bfloat16_rn(r2);
    hi = __bfloat16_as_ushort(h);
    mid = __bfloat16_as_ushort(m);
    lo = __bfloat16_as_ushort(l);
}


// A tile is refined in PASSES over the whole sequence set: EM iteration `it` (0-based) is one EM pass (E-step fused
// with the M-step counts), the last pass is the final E-step (refine.hpp:306).  Every role decodes the same list.
//
// The exponentials of an EM pass are taken relative to ONE reference per bucket and pass, tc_ref_below(l) = 64 ... 108
// under the upper bound ub = sum_c max_r D[c][r] of every window weight of the model: e = 2^(w - ub + 108) <= 2^108 cannot overflow
// (nor can a sequence's sum, or the FP32 count accumulators), and a sequence whose best window lies up to
// offset + 100 below ub (l = 20: seven columns at the 1e-9 floor) still has its leading terms 24 binades above the FP32
// underflow threshold; relative precision does not depend on the scale.  A sequence below that range (its sum under
// kTcMinSum) flags the bucket for the exact kernel.  This replaces the separate per-sequence maximum passes
// (GEMM1 + a max scan of S) that the first two iterations needed to find a reference.
enum : int { kTcPassEm = 1, kTcPassFinal = 2 };
constexpr float kTcRefBelow = 108.f;                 // log2 units, at l = 20 (tc_ref_below)
constexpr float kTcMinSum = 7.888609052210118e-31f;  // 2^-100
// How far under the bound the reference sits.  The FP32 accumulators of GEMM1 hold weight - reference, so their
// rounding error (a few ulps of that magnitude) grows with the offset: measured max |d theta| against the reference on
// random sets 1.7e-5 / 3.5e-5 / 7.6e-5 at 32 / 64 / 108.  What the offset buys is range -- a sequence whose best window
// lies more than offset + 100 under the bound flags its bucket -- and the depth a sequence can sink to grows with the
// motif length (one column at the 1e-9 floor costs 28): at l = 20 an offset of 64 flags 2.5 x as many buckets as 108,
// at l <= 16 it flags fewer (better precision, fewer near-ties).  Hence 64 up to l = 16 and 11 more per extra column.
__host__ __device__ inline float tc_ref_below(int l) { return l <= 16 ? 64.f : fminf(kTcRefBelow, 64.f + 11.f * static_cast<float>(l - 16)); }
struct TcPass {
    int kind, it;
    bool new_model;  // theta -> log-odds terms are rebuilt before this pass (always: every pass has its own model)
};
__device__ __forceinline__ int tc_num_passes(int max_iters) { return max_iters + 1; }
__device__ __forceinline__ TcPass tc_pass(int ps, int max_iters) {
    TcPass r;
    r.it = ps;
    r.kind = ps < max_iters ? kTcPassEm : kTcPassFinal;
    r.new_model = true;
    return r;
}

// number of shared-memory bytes the kernel needs (mirrored by the carve-up below)
__host__ __device__ inline size_t tc_smem_bytes(int t, int n_blocks, int e_positions) {
    size_t b = 0;
    b += static_cast<size_t>(4) * e_positions * 8;                 // E0/E1 of two sequences
    b += static_cast<size_t>(t) * kTcRows * 4;                       // argmax of every sequence (final pass)
    b += static_cast<size_t>(2) * 2 * kTcRows * 16;                  // partner exchange, double-buffered
    b += static_cast<size_t>(n_blocks) * sizeof(TcBlock);
    b += static_cast<size_t>(t) * 16 + 16;                           // per-sequence metadata (+ win_off[t])
    b += 32 * 8;                                                     // mbarriers, tmem slot
    return b + 128;
}

#ifdef PM_TC_TIMING
// clock sums of CTA 0 into p.phase_clk: [0] softmax thread total [1] its wait for S blocks [2] for the counts of a
// sequence [3] model updates [4] MMA thread: wait for P blocks [5] for one-hot arrays [6] for models / count buffers
// [7] MMA thread total
#define TC_T0() const long long tc_t0_ = clock64()
#define TC_ACC(var) var += clock64() - tc_t0_
#else
#define TC_T0() do {} while (0)
#define TC_ACC(var) do {} while (0)
#endif

// ---------------------------------------------------------------------------------------------------------
// the kernel
// ---------------------------------------------------------------------------------------------------------
template <int KC>  // base positions covered by K = 4 KC (multiple of 16): KC = 4 ceil(l / 4)
__global__ void __launch_bounds__(kTcThreads, 1) em_refine_tc_kernel(const EmParams p, const TcExtra x) {
    constexpr int K = 4 * KC;
    constexpr int NBLK = KC <= 16 ? 128 : 96;
    constexpr int HP = KC / 2;  // base positions per warpgroup
    // tensor-memory columns
    constexpr uint32_t cD = 0;             // 3 terms x 2 KC
    constexpr uint32_t cO = 6 * KC;        // 2 buffers x 4 KC
    constexpr uint32_t cS = 14 * KC;       // 2 buffers x NBLK
    static_assert(cS + 2 * NBLK <= 512, "tensor memory budget");

    extern __shared__ __align__(128) unsigned char smem[];
    const int t = p.t, l = p.l;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    {
        const unsigned int n_all = p.n_work_dev ? *p.n_work_dev : p.n_work;
        if (n_all < x.min_work) {  // small batch: nothing is decided here
            for (unsigned int i = blockIdx.x * blockDim.x + tid; i < n_all; i += gridDim.x * blockDim.x) x.out_flag[i] = kTcFlagSmall;
            return;
        }
    }
    const int EB = x.e_positions * 8;  // bytes per one-hot array
    unsigned char* Ebuf = smem;        // [2 sequences][2 parities][EB]
    float* mprev = reinterpret_cast<float*>(Ebuf + 4 * static_cast<size_t>(EB));  // [t][128]: the final pass's argmax per sequence
    float4* xch = reinterpret_cast<float4*>(mprev + static_cast<size_t>(t) * kTcRows);  // [2][2][128]
    TcBlock* blocks = reinterpret_cast<TcBlock*>(xch + 2 * 2 * kTcRows);
    int* smeta = reinterpret_cast<int*>(blocks + x.n_blocks);  // [t][4]: first word (global index), windows, first flat index, bases
    unsigned long long* bars = reinterpret_cast<unsigned long long*>((reinterpret_cast<uintptr_t>(smeta + 4 * t + 4) + 7) & ~static_cast<uintptr_t>(7));
    unsigned long long* e_full = bars;        // [2]
    unsigned long long* e_empty = bars + 2;   // [2]
    unsigned long long* s_full = bars + 4;    // [2]
    unsigned long long* p_full = bars + 6;    // [2]
    unsigned long long* o_full = bars + 8;    // [2]
    unsigned long long* o_free = bars + 10;   // [2]
    unsigned long long* d_full = bars + 12;   // [1]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 14);

    for (int i = tid; i < x.n_blocks * static_cast<int>(sizeof(TcBlock) / 4); i += blockDim.x)
        reinterpret_cast<uint32_t*>(blocks)[i] = reinterpret_cast<const uint32_t*>(x.blocks)[i];
    for (int i = tid; i < t; i += blockDim.x) {
        smeta[4 * i + 0] = static_cast<int>(p.word_off[i]);
        smeta[4 * i + 1] = p.seq_len[i] - l + 1;
        smeta[4 * i + 2] = static_cast<int>(p.win_off[i]);
        smeta[4 * i + 3] = p.seq_len[i];
    }
    if (tid == 0) {
        for (int b = 0; b < 2; ++b) {
            mbar_init(&e_full[b], 1);
            mbar_init(&e_empty[b], 1);
            mbar_init(&s_full[b], 1);
            mbar_init(&p_full[b], kTcSoftWarps);
            mbar_init(&o_full[b], 1);
            mbar_init(&o_free[b], kTcSoftWarps);
        }
        mbar_init(&d_full[0], kTcSoftWarps);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 8) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)), "r"(512u) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    const unsigned int n_work = p.n_work_dev ? *p.n_work_dev : p.n_work;
    const unsigned int n_tiles = (n_work + kTcRows - 1) / kTcRows;
    const int n_passes = tc_num_passes(p.max_iters);
    const int NB = x.n_blocks;

    // Register budget by role.  The register file is per sub-partition, 3 warps x 168 registers at launch: the third
    // warpgroup keeps 72 per thread and the softmax warpgroups take 216 (2 x 216 + 72 = 3 x 168, the pool is what the
    // CTA was launched with), which holds a chunk of S, the outgoing P chunk and the count accumulators without spills.
    // Each setmaxnreg sits inside its role's branch so that the assembler can tell which limit the code below runs under.
    if (warp >= 10) {
        // idle: these warps only complete the third warpgroup (setmaxnreg is a warpgroup-wide instruction)
        asm volatile("setmaxnreg.dec.sync.aligned.u32 72;");
    } else if (warp == 9) {
        asm volatile("setmaxnreg.dec.sync.aligned.u32 72;");
        // ================= producer: one-hot codes of the next sequence =================
        // The arrays depend on the sequence only, so the producer simply cycles through the set; every sweep of
        // every tile consumes the sequences in the same order.
        unsigned int sq = 0;
        for (unsigned int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
            for (int ps = 0; ps < n_passes; ++ps) {
                for (int i = 0; i < t; ++i, ++sq) {
                    tc_wait(&e_empty[sq & 1], ((sq >> 1) & 1) ^ 1);
                    unsigned char* E0 = Ebuf + static_cast<size_t>(sq & 1) * 2 * EB;
                    unsigned char* E1 = E0 + EB;
                    const uint64_t* __restrict__ wp = p.words + smeta[4 * i];
                    const int n = smeta[4 * i + 3];
                    for (int q0 = 0; q0 < x.e_positions; q0 += 32) {
                        const int q = q0 + lane;
                        // base q (array 0) and base q + 1 (array 1, the odd windows)
                        const uint64_t w0 = q0 < n ? wp[q0 >> 5] : 0ULL;
                        const uint64_t w1 = q0 + 32 < n ? wp[(q0 >> 5) + 1] : 0ULL;
                        const unsigned s0 = static_cast<unsigned>(w0 >> (62 - 2 * lane)) & 3u;
                        const unsigned s1 = lane < 31 ? static_cast<unsigned>(w0 >> (60 - 2 * lane)) & 3u : static_cast<unsigned>(w1 >> 62) & 3u;
                        const uint64_t c0 = q < n ? (0x3F80ULL << (16 * s0)) : 0ULL;
                        const uint64_t c1 = q + 1 < n ? (0x3F80ULL << (16 * s1)) : 0ULL;
                        if (q < x.e_positions) {
                            *reinterpret_cast<uint64_t*>(E0 + 8 * q) = c0;
                            *reinterpret_cast<uint64_t*>(E1 + 8 * q) = c1;
                        }
                    }
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    __syncwarp();
                    if (lane == 0) tc_mbar_arrive(&e_full[sq & 1]);
                }
            }
        }
    } else if (warp == 8) {
        asm volatile("setmaxnreg.dec.sync.aligned.u32 72;");
        // ================= MMA issuer: the warp stays converged, one elected lane issues =================
        {
            constexpr uint32_t idesc_base = (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(kTcRows >> 4) << 24);
            constexpr uint32_t idesc2 = idesc_base | (1u << 16) | (static_cast<uint32_t>(K >> 3) << 17);
            constexpr uint32_t hi1 = (128u >> 4) | (1u << 14);  // SBO = 128 B, descriptor version 1
            constexpr uint32_t hi2 = (16u >> 4) | (1u << 14);   // SBO = 16 B
            const uint32_t e_addr = smem_u32(Ebuf) >> 4;
            const uint32_t eb16 = static_cast<uint32_t>(EB) >> 4;
            unsigned int blk = 0, sq_g1 = 0, sq_g2 = 0, oq = 0, sw = 0;
            long long tm_p = 0, tm_e = 0, tm_d = 0;
            const long long tm_begin = clock64();

            auto issue_g1 = [&](const TcBlock& B, unsigned int buf, unsigned int sq) {
                const uint32_t tS = tmem + cS + buf * NBLK;
#pragma unroll 1
                for (int sgi = 0; sgi < 2; ++sgi) {
                    const TcSeg sg = B.seg[sgi];
                    if (sg.n == 0) continue;
                    const uint32_t lo = ((e_addr + ((sq & 1) * 2 + sg.par) * eb16 + sg.i0) & 0x3FFFu) | (1u << 16);  // LBO = 16 B
                    const uint32_t idesc = idesc_base | (static_cast<uint32_t>(sg.n >> 3) << 17);
                    const uint32_t d = tS + sg.col;
                    if (tc_elect()) {
#pragma unroll
                        for (int kb = 0; kb < KC / 4; ++kb) tc_mma(d, tmem + cD + 8 * kb, lo + 2 * kb, hi1, idesc, kb != 0);
#pragma unroll
                        for (int term = 1; term < 3; ++term) {
#pragma unroll
                            for (int kb = 0; kb < KC / 4; ++kb) tc_mma(d, tmem + cD + term * 2 * KC + 8 * kb, lo + 2 * kb, hi1, idesc, true);
                        }
                    }
                    __syncwarp();
                }
                if (tc_elect()) tc_commit(&s_full[buf]);
                __syncwarp();
            };

            for (unsigned int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
                for (int ps = 0; ps < n_passes; ++ps) {
                    const TcPass pass = tc_pass(ps, p.max_iters);
                    const bool with_counts = pass.kind == kTcPassEm;  // otherwise GEMM1 only
                    if (pass.new_model) {
                        TC_T0();
                        tc_wait(&d_full[0], sw & 1);
                        TC_ACC(tm_d);
                        ++sw;
                        tc_fence_after();
                    }
                    // first block of the sweep
                    {
                        TC_T0();
                        tc_wait(&e_full[sq_g1 & 1], (sq_g1 >> 1) & 1);
                        TC_ACC(tm_e);
                    }
                    issue_g1(blocks[0], blk & 1, sq_g1);
                    if (blocks[0].last) ++sq_g1;
                    bool o_acc = false;
#pragma unroll 1
                    for (int n = 0; n < NB; ++n, ++blk) {
                        const TcBlock B = blocks[n];
                        if (n + 1 < NB) {
                            const TcBlock& B1 = blocks[n + 1];
                            if (B1.first) {
                                TC_T0();
                                tc_wait(&e_full[sq_g1 & 1], (sq_g1 >> 1) & 1);
                                TC_ACC(tm_e);
                            }
                            issue_g1(B1, (blk + 1) & 1, sq_g1);
                            if (B1.last) ++sq_g1;
                        }
                        {
                            TC_T0();
                            tc_wait(&p_full[blk & 1], (blk >> 1) & 1);
                            TC_ACC(tm_p);
                        }
                        tc_fence_after();
                        if (with_counts) {
                            if (B.first) {
                                TC_T0();
                                tc_wait(&o_free[oq & 1], ((oq >> 1) & 1) ^ 1);
                                TC_ACC(tm_d);
                                tc_fence_after();
                                o_acc = false;
                            }
                            const uint32_t tS = tmem + cS + (blk & 1) * NBLK;
                            const uint32_t tO = tmem + cO + (oq & 1) * K;
#pragma unroll 1
                            for (int sgi = 0; sgi < 2; ++sgi) {
                                const TcSeg sg = B.seg[sgi];
                                const uint32_t lo0 = ((e_addr + ((sq_g2 & 1) * 2 + sg.par) * eb16 + sg.i0) & 0x3FFFu) | ((128u >> 4) << 16);  // LBO = 128 B
                                if (tc_elect()) {
#pragma unroll 1
                                    for (int c = 0; c < sg.valid; c += 16) {
                                        const uint32_t a = tS + sg.col + c;
                                        tc_mma(tO, a, lo0 + c, hi2, idesc2, o_acc || c > 0);
                                        tc_mma(tO, a + 8, lo0 + c, hi2, idesc2, true);
                                    }
                                }
                                __syncwarp();
                                if (sg.valid > 0) o_acc = true;
                            }
                            if (B.last) {
                                if (tc_elect()) tc_commit(&o_full[oq & 1]);
                                __syncwarp();
                                ++oq;
                            }
                        }
                        if (B.last) {
                            if (tc_elect()) tc_commit(&e_empty[sq_g2 & 1]);
                            __syncwarp();
                            ++sq_g2;
                        }
                    }
                }
            }
            (void)tm_p; (void)tm_e; (void)tm_d; (void)tm_begin;
        }
        __syncwarp();
    } else {
        // ================= softmax warpgroups: thread = bucket row, warpgroup = column half =================
        asm volatile("setmaxnreg.inc.sync.aligned.u32 216;");
        const int row = tid & 127, wg = tid >> 7;
        const uint32_t lane_base = static_cast<uint32_t>((warp & 3) * 32) << 16;
        const uint32_t tD = tmem + lane_base + cD, tO = tmem + lane_base + cO, tS = tmem + lane_base + cS;
        const int c_lo = wg * HP;  // my base positions [c_lo, c_lo + HP)
        constexpr float kLn2 = 0.6931471805599453f;
        double sum_logw = 0.0;
        for (int i = 0; i < t; ++i) sum_logw += p.seq_logw[i];

        unsigned int blk = 0, oq = 0, xq = 0;
        [[maybe_unused]] long long ts_s = 0, ts_o = 0, ts_u = 0, ts_kind[3] = {0, 0, 0}, ts_close = 0;
        [[maybe_unused]] const long long ts_begin = clock64();
        for (unsigned int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
            const unsigned int wi = tile * kTcRows + row;
            const bool live = wi < n_work;
            const WorkDesc wd = live ? p.work[wi] : WorkDesc{0, 0, 0, 0};
            float acc[4 * HP];       // my columns' expected counts (EM sweeps) / theta0 counts
            unsigned flags = 0;
            double ref_eff = 0.0;  // reference of the current pass's exponentials (log2 units), as GEMM1 subtracts it
            double prev_ll = 0.0, expct = 0.0;
            double lbg[4];           // natural logs of the current background column

            // ---- init_model (refine.hpp:90-127), pseudocount 0: integer symbol counts of the members
            {
                uint32_t cnt8[HP];
#pragma unroll
                for (int c = 0; c < HP; ++c) cnt8[c] = 0;
                for (unsigned int m = 0; m < wd.count; ++m) {
                    const int64_t f = p.members[wd.mem_begin + m];
                    int i = 0;
                    for (int hi = t; hi - i > 1;) {
                        const int mid = (i + hi) >> 1;
                        if (smeta[4 * mid + 2] <= f) i = mid; else hi = mid;
                    }
                    const uint64_t v = load_window(p.words + smeta[4 * i], f - smeta[4 * i + 2]);
#pragma unroll
                    for (int c = 0; c < HP; ++c) cnt8[c] += 1u << (8 * (static_cast<unsigned>(v >> (62 - 2 * (c_lo + c))) & 3u));
                }
                const float inv_n = wd.count ? 1.f / static_cast<float>(wd.count) : 0.f;
#pragma unroll
                for (int c = 0; c < HP; ++c) {
#pragma unroll
                    for (int r = 0; r < 4; ++r) acc[4 * c + r] = static_cast<float>((cnt8[c] >> (8 * r)) & 255u) * inv_n;
                }
                // log of the global symbol frequencies (theta0's background column)
                for (int r = 0; r < 4; ++r) lbg[r] = log(fmax(p.tot_sym[r] / p.tot_bases, 1e-9));
            }

            for (int ps = 0; ps < n_passes; ++ps) {
                const TcPass pass = tc_pass(ps, p.max_iters);
                const bool final_sweep = pass.kind == kTcPassFinal, em_pass = pass.kind == kTcPassEm;
                // ---- theta of this iteration -> log-odds terms in tensor memory.  Iteration 0: acc holds theta0 itself;
                // otherwise acc holds the expected counts of the previous EM pass (M-step, refine.hpp:227-269).
                if (pass.new_model) {
                    TC_T0();
                    if (pass.it > 0) {
                        // background = symbol totals - expected motif counts, clamped at 0 (refine.hpp:241-253)
                        float part[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
                        for (int c = 0; c < HP; ++c) {
                            if (c_lo + c < l) {
#pragma unroll
                                for (int r = 0; r < 4; ++r) part[r] += acc[4 * c + r];
                            }
                        }
                        const float4 mine = make_float4(part[0], part[1], part[2], part[3]);
                        xch[(xq & 1) * 2 * kTcRows + wg * kTcRows + row] = mine;
                        tc_named_sync();
                        const float4 oth = xch[(xq & 1) * 2 * kTcRows + (wg ^ 1) * kTcRows + row];
                        ++xq;
                        // fixed order (warpgroup 0 first) so both partners compute identical values
                        const float4 a4 = wg == 0 ? mine : oth, b4 = wg == 0 ? oth : mine;
                        double raw[4] = {fmax(p.tot_sym[0] - (static_cast<double>(a4.x) + static_cast<double>(b4.x)), 0.0),
                                         fmax(p.tot_sym[1] - (static_cast<double>(a4.y) + static_cast<double>(b4.y)), 0.0),
                                         fmax(p.tot_sym[2] - (static_cast<double>(a4.z) + static_cast<double>(b4.z)), 0.0),
                                         fmax(p.tot_sym[3] - (static_cast<double>(a4.w) + static_cast<double>(b4.w)), 0.0)};
                        const double sum = raw[0] + raw[1] + raw[2] + raw[3];
                        double fs = 0.0;
#pragma unroll
                        for (int r = 0; r < 4; ++r) {
                            raw[r] = sum > 0.0 ? fmax(raw[r] / sum, 1e-9) : 0.25;
                            fs += raw[r];
                        }
#pragma unroll
                        for (int r = 0; r < 4; ++r) {
                            const double tv = raw[r] / fs;
                            lbg[r] = log(fmax(tv, 1e-9));
                            if (p.out_theta && live && wg == 0 && final_sweep)
                                p.out_theta[static_cast<int64_t>(wi) * 4 * (l + 1) + r * (l + 1)] = tv;
                        }
                    }
                    // per column: write_column (refine.hpp:256-269), expectation = sum_c max_r theta[r][c]
                    // (refine.hpp:130-136) and the log-odds D[c][r] = log2 max(theta,1e-9) - log2 max(bg,1e-9).  FP32
                    // throughout: the counts are FP32 sums; log2f is accurate to 1 ulp (2e-6 at |D| = 20).
                    float ex_part = 0.f, ub_part = 0.f;
                    float dval[4 * HP];
                    float lbg2[4];
#pragma unroll
                    for (int r = 0; r < 4; ++r) lbg2[r] = static_cast<float>(lbg[r] * 1.4426950408889634);
#pragma unroll
                    for (int c = 0; c < HP; ++c) {
                        const bool col_live = c_lo + c < l;
                        float v[4];
                        if (pass.it > 0) {
                            const float cs = (acc[4 * c] + acc[4 * c + 1]) + (acc[4 * c + 2] + acc[4 * c + 3]);
                            const float ics = 1.f / cs;
                            float f2 = 0.f;
#pragma unroll
                            for (int r = 0; r < 4; ++r) {
                                v[r] = cs > 0.f ? fmaxf(acc[4 * c + r] * ics, 1e-9f) : 0.25f;
                                f2 += v[r];
                            }
                            const float if2 = 1.f / f2;
#pragma unroll
                            for (int r = 0; r < 4; ++r) v[r] *= if2;
                        } else {
#pragma unroll
                            for (int r = 0; r < 4; ++r) v[r] = acc[4 * c + r];
                        }
                        float mx = 0.f;
#pragma unroll
                        for (int r = 0; r < 4; ++r) {
                            mx = fmaxf(mx, v[r]);
                            dval[4 * c + r] = col_live ? log2f(fmaxf(v[r], 1e-9f)) - lbg2[r] : 0.f;
                            if (p.out_theta && live && col_live && final_sweep)
                                p.out_theta[static_cast<int64_t>(wi) * 4 * (l + 1) + r * (l + 1) + (c_lo + c + 1)] = static_cast<double>(v[r]);
                        }
                        if (col_live) ex_part += mx;
                        ub_part += fmaxf(fmaxf(dval[4 * c], dval[4 * c + 1]), fmaxf(dval[4 * c + 2], dval[4 * c + 3]));  // dead columns: all zero
                    }
                    // expectation and the weight bound: partner exchange
                    xch[(xq & 1) * 2 * kTcRows + wg * kTcRows + row] = make_float4(ex_part, ub_part, 0.f, 0.f);
                    tc_named_sync();
                    float qref;  // what every live column gives up so that GEMM1 delivers weight minus reference
                    {
                        const float4 oth = xch[(xq & 1) * 2 * kTcRows + (wg ^ 1) * kTcRows + row];
                        ++xq;
                        expct = wg == 0 ? static_cast<double>(ex_part) + static_cast<double>(oth.x) : static_cast<double>(oth.x) + static_cast<double>(ex_part);
                        const float ub = wg == 0 ? ub_part + oth.y : oth.y + ub_part;  // same value in both partners
                        // The reference of this pass's exponentials, tc_ref_below(l) under the bound, is folded into the
                        // log-odds: every window has exactly l live columns, so taking ref / l off every entry makes
                        // GEMM1 produce weight - ref itself (one subtraction per element less in the sweep).  The final
                        // E-step only compares weights: the shift does not matter there.
                        qref = (ub - tc_ref_below(l)) / static_cast<float>(l);
                        ref_eff = static_cast<double>(l) * static_cast<double>(qref);
                    }
                    // three bf16 terms (hi + mid + lo = 24 significant bits) of D - ref / l
                    uint32_t dcol[3][2 * HP];
#pragma unroll
                    for (int c = 0; c < HP; ++c) {
                        const bool col_live = c_lo + c < l;
                        uint32_t h[4], m[4], lw[4];
#pragma unroll
                        for (int r = 0; r < 4; ++r) tc_split3(col_live ? dval[4 * c + r] - qref : 0.f, h[r], m[r], lw[r]);
                        dcol[0][2 * c] = h[0] | (h[1] << 16);
                        dcol[0][2 * c + 1] = h[2] | (h[3] << 16);
                        dcol[1][2 * c] = m[0] | (m[1] << 16);
                        dcol[1][2 * c + 1] = m[2] | (m[3] << 16);
                        dcol[2][2 * c] = lw[0] | (lw[1] << 16);
                        dcol[2][2 * c + 1] = lw[2] | (lw[3] << 16);
                    }
#pragma unroll
                    for (int term = 0; term < 3; ++term) {
#pragma unroll
                        for (int q = 0; q < 2 * HP; q += 4) tc_st4(tD + term * 2 * KC + 2 * c_lo + q, &dcol[term][q]);
                    }
                    tc_wait_st();
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) tc_mbar_arrive(&d_full[0]);
#pragma unroll
                    for (int e = 0; e < 4 * HP; ++e) acc[e] = 0.f;
                    TC_ACC(ts_u);
                }

                // ---- the sweep: every sequence, block by block
#ifdef PM_TC_TIMING
                const long long ts_pass0 = clock64();
#endif
                double ll = 0.0;
                TcSeqState st = {-INFINITY, -INFINITY, 0};
                bool pending = false;   // the previous sequence's O block has not been folded into acc yet
                unsigned int pend_oq = 0;
                // Folds the counts of the sequence whose GEMM2 has finished into acc.  Its normaliser needs no sum in the
                // softmax threads: every window has a base under motif column 0, so the four symbol counts of that column
                // add up to sum_j e_j = L -- read from the same accumulator (by both partners: four more columns), made of
                // the very hi + lo terms the counts are made of, so the normalised counts of a column sum to one exactly.
                auto fold_pending = [&]() {
                    {
                        TC_T0();
                        tc_wait(&o_full[pend_oq & 1], (pend_oq >> 1) & 1);
                        TC_ACC(ts_o);
                    }
                    tc_fence_after();
                    const uint32_t base = tO + (pend_oq & 1) * K;
                    const uint32_t src = base + 4 * c_lo;
                    uint32_t r0[4];
                    tc_ld4(base, r0);
                    uint32_t r[4 * HP];
#pragma unroll
                    for (int q = 0; q < 4 * HP; q += 16) {
                        if (q + 16 <= 4 * HP) {
                            tc_ld16(src + q, r + q);
                        } else {
#pragma unroll
                            for (int q4 = q; q4 < 4 * HP; q4 += 4) tc_ld4(src + q4, r + q4);
                        }
                    }
                    tc_wait_ld();
                    const float L = (__uint_as_float(r0[0]) + __uint_as_float(r0[1])) + (__uint_as_float(r0[2]) + __uint_as_float(r0[3]));
                    // below kTcMinSum the sequence's best window is more than offset + 100 under the bound: out of range
                    if (!(L >= kTcMinSum) || !(L < INFINITY)) flags |= kTcFlagRange;
                    const float inv = 1.f / L;
#pragma unroll
                    for (int e = 0; e < 4 * HP; ++e) acc[e] = fmaf(__uint_as_float(r[e]), inv, acc[e]);
                    if (wg == 0) {
                        // log2 L = exponent + log2(mantissa): the absolute error stays at 1e-7 whatever the scale
                        const uint32_t lb = __float_as_uint(L);
                        const float mant = __uint_as_float((lb & 0x007FFFFFu) | 0x3F800000u);
                        const int ex = static_cast<int>(lb >> 23) - 127;
                        ll += ((ref_eff + static_cast<double>(ex)) + static_cast<double>(log2f(mant))) * 0.6931471805599453;
                    }
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) tc_mbar_arrive(&o_free[pend_oq & 1]);
                    pending = false;
                };

#pragma unroll 1
                for (int n = 0; n < NB; ++n, ++blk) {
                    const TcBlock B = blocks[n];
                    const int i = B.seq;
                    if (B.first) {
                        st.mxa = -INFINITY;
                        st.second = -INFINITY;
                        st.best_j = 0;
                    }
                    {
                        TC_T0();
                        tc_wait(&s_full[blk & 1], (blk >> 1) & 1);
                        TC_ACC(ts_s);
                    }
                    tc_fence_after();
                    const uint32_t tB = tS + (blk & 1) * NBLK;
                    const int half = B.ncols >> 1;
                    const int c_begin = wg * half, c_end = c_begin + half;
#pragma unroll 1
                    for (int sgi = 0; sgi < 2; ++sgi) {
                        // my columns of this segment: [lo, hi), of which those below vend are real windows
                        const TcSeg sg = B.seg[sgi];
                        const int lo = max(c_begin, static_cast<int>(sg.col)), hi = min(c_end, sg.col + sg.n);
                        const int vend = min(hi, sg.col + sg.valid);
                        int cc = lo;
                        int j = 2 * (sg.i0 + lo - sg.col) + sg.par;
#pragma unroll 1
                        for (; cc + 32 <= vend; cc += 32, j += 64) {  // two full chunks: no masks
                            uint32_t r[32];
                            tc_ld32(tB + cc, r);
                            tc_wait_ld();
                            if (em_pass) {
                                uint32_t o[32];
                                tc_em_chunk<false>(r, o, 16);
                                tc_em_chunk<false>(r + 16, o + 16, 16);
                                tc_st32(tB + cc, o);
                            } else {
                                tc_final_chunk<false>(r, 16, j, st);
                                tc_final_chunk<false>(r + 16, 16, j + 32, st);
                            }
                        }
#pragma unroll 1
                        for (; cc < vend; cc += 16, j += 32) {  // at most one full chunk and the tail (dead chunks are skipped)
                            const int nv = min(vend - cc, 16);
                            uint32_t r[16];
                            tc_ld16(tB + cc, r);
                            tc_wait_ld();
                            if (em_pass) {
                                uint32_t o[16];
                                tc_em_chunk<true>(r, o, nv);
                                tc_st16(tB + cc, o);
                            } else {
                                tc_final_chunk<true>(r, nv, j, st);
                            }
                        }
                    }
                    if (em_pass) tc_wait_st();
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) tc_mbar_arrive(&p_full[blk & 1]);

                    if (pending) fold_pending();  // the previous sequence's counts: its GEMM2 finished long ago

                    if (B.last && em_pass) {
                        // nothing to exchange: the normaliser comes out of GEMM2 (fold_pending)
                        pend_oq = oq++;
                        pending = true;
                    } else if (B.last) {
                        TC_T0();
                        // ---- close the sequence (final pass): both column halves -> maximum, its window, runner-up
                        float4 mine = make_float4(0.f, st.mxa, st.second, __int_as_float(tc_final_window(st)));
                        xch[(xq & 1) * 2 * kTcRows + wg * kTcRows + row] = mine;
                        tc_named_sync();
                        const float4 oth = xch[(xq & 1) * 2 * kTcRows + (wg ^ 1) * kTcRows + row];
                        ++xq;
                        const float4 a4 = wg == 0 ? mine : oth, b4 = wg == 0 ? oth : mine;  // fixed order
                        if (wg == 0) {
                            // argmax with margin: the runner-up must lie tie_delta below the maximum (ties go to the
                            // smallest offset in the reference, refine.hpp:311-316: decided by the exact kernel)
                            const float M = fmaxf(a4.y, b4.y);
                            if (!(M > -INFINITY) || !(M < INFINITY)) flags |= kTcFlagBad;
                            const float sec = fmaxf(fmaxf(a4.z, b4.z), fminf(a4.y, b4.y));
                            const int bj = a4.y >= b4.y ? __float_as_int(a4.w) : __float_as_int(b4.w);
                            // the weights compared here carry their column number in the low mantissa bits
                            // and are weight minus reference; the relative part of the margin scales with the weight itself
                            // (the accumulation error of GEMM1, ~1e-5 at these magnitudes, is far inside the absolute part)
                            const float m_raw = M + static_cast<float>(ref_eff);
                            const float delta2 = (x.tie_delta + 1e-5f * fabsf(m_raw * kLn2)) * kLog2e + kTcFinalUlpMargin * fabsf(M);
                            if (!(M - sec > delta2)) flags |= kTcFlagTie;
                            if (live && p.out_pos) p.out_pos[static_cast<int64_t>(wi) * t + i] = bj + 1;
                            // parked for the profile below
                            mprev[i * kTcRows + row] = __int_as_float(bj);
                        }
                        TC_ACC(ts_close);
                    }
                }
                if (pending) fold_pending();
#ifdef PM_TC_TIMING
                ts_kind[pass.kind] += clock64() - ts_pass0;
#endif

                if (em_pass) {
                    // ---- log-likelihood of the model that entered this iteration and the stop test (refine.hpp:296-304)
                    if (wg == 0) {
                        double llv = ll - sum_logw;
                        for (int r = 0; r < 4; ++r) llv += p.tot_sym[r] * lbg[r];
                        const int it = pass.it + 1;
                        if (p.out_ll && live) p.out_ll[static_cast<int64_t>(wi) * p.max_iters + pass.it] = llv;
                        // iterations 2 .. max_iters-1 can stop the loop; a gain that is not clearly above tol is not
                        // decided with FP32 sums
                        if (it >= 2 && it < p.max_iters && !(llv - prev_ll >= p.tol + static_cast<double>(x.ll_margin))) flags |= kTcFlagConv;
                        if (!(llv == llv)) flags |= kTcFlagBad;
                        prev_ll = llv;
                    }
                } else if (final_sweep && wg == 0 && live) {
                    // ---- score / consensus over the argmax rows (scoring.hpp:84-126)
                    uint32_t prof8[KC];  // symbol counts of the argmax rows, one byte per symbol
#pragma unroll
                    for (int c = 0; c < KC; ++c) prof8[c] = 0;
                    for (int i = 0; i < t; ++i) {
                        const uint64_t v = load_window(p.words + smeta[4 * i], __float_as_int(mprev[i * kTcRows + row]));
#pragma unroll
                        for (int c = 0; c < KC; ++c) prof8[c] += 1u << (8 * (static_cast<unsigned>(v >> (62 - 2 * c)) & 3u));
                    }
                    int score = 0;
                    unsigned long long cons = 0ULL;
#pragma unroll
                    for (int c = 0; c < KC; ++c) {
                        if (c < l) {
                            int best = 0, bv = static_cast<int>(prof8[c] & 255u);
#pragma unroll
                            for (int r = 1; r < 4; ++r) {
                                const int v = static_cast<int>((prof8[c] >> (8 * r)) & 255u);
                                if (v > bv) {
                                    bv = v;
                                    best = r;
                                }
                            }
                            score += bv;
                            cons |= static_cast<unsigned long long>(best) << (62 - 2 * c);
                        }
                    }
                    p.out_score[wi] = score;
                    p.out_iters[wi] = p.max_iters;
                    p.out_exp[wi] = expct;
                    p.out_cons[wi] = cons;
                    x.out_flag[wi] = static_cast<unsigned char>(flags);
                    if (flags == 0) {
                        atomicAdd(p.iter_total, static_cast<unsigned long long>(p.max_iters + 1));
                    } else {
                        if (flags & kTcFlagConv) atomicAdd(&x.stats[0], 1ULL);
                        if (flags & kTcFlagRange) atomicAdd(&x.stats[1], 1ULL);
                        if (flags & kTcFlagTie) atomicAdd(&x.stats[2], 1ULL);
                        if (flags & kTcFlagBad) atomicAdd(&x.stats[3], 1ULL);
                    }
                }
            }
        }
#ifdef PM_TC_TIMING
        if (blockIdx.x == 0 && tid == 0) {
            atomicAdd(p.phase_clk + 0, static_cast<unsigned long long>(clock64() - ts_begin));
            atomicAdd(p.phase_clk + 1, static_cast<unsigned long long>(ts_s));
            atomicAdd(p.phase_clk + 2, static_cast<unsigned long long>(ts_o));
            atomicAdd(p.phase_clk + 3, static_cast<unsigned long long>(ts_u));
            atomicAdd(p.phase_clk + 4, static_cast<unsigned long long>(ts_kind[kTcPassEm]));
            atomicAdd(p.phase_clk + 5, static_cast<unsigned long long>(ts_kind[0]));
            atomicAdd(p.phase_clk + 6, static_cast<unsigned long long>(ts_kind[kTcPassFinal]));
            atomicAdd(p.phase_clk + 7, static_cast<unsigned long long>(ts_close));
        }
#endif
    }

    tc_fence_before();
    __syncthreads();
    if (warp == 8) {
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512u) : "memory");
    }
}

}  // namespace k
}  // namespace pm
