// pm_em_pair.cuh — EM refinement, TWO enriched buckets per CTA in lockstep: the EM kernel of every set whose
// sequences fit a tile (small sets such as the t=20 configurations of BASELINE.json keep all per-sequence state
// and the whole packed set in shared memory; large sets walk the tiles, see `big` below).
//
// Same algorithm, precision scheme and tile/class-group index as pm_em_smem.cuh (refine.hpp:90-326); what
// changes is that everything that depends on the SEQUENCE SET only is done once for two buckets:
//   * the window word assembly and the nibble offsets of the E-step: one LDS.64 fetches the pair-table
//     entries {T_A[g][q], T_B[g][q]} of both buckets (16 entries x 8 B = all 32 banks, conflict-free);
//   * the responsibilities are stored interleaved {z_A[j], z_B[j]} so the M-step's class-row entry (slot of
//     the base position) is loaded once and each LDS.64 of the gather feeds both buckets' accumulators
//     (rows built for distinct slots mod 32 are also conflict-free for 8-byte slots: each half-warp covers
//     the 32 banks exactly once);
//   * the arithmetic on the two buckets' values uses the packed FP32x2 instructions of sm_100 (FADD2, FMUL2,
//     FFMA2): one instruction per pair, same round-to-nearest results;
//   * loop control, prefetch of the class rows, sequence metadata.
// Instruction count per bucket is less than half of the one-bucket kernel's; shared-memory wavefronts per
// bucket stay the same (8 per 32 windows in the E-step, 8 per class row in the M-step), which is the bound.
//
// Buckets of a pair iterate in lockstep.  A bucket whose likelihood gain fell below tol (refine.hpp:300) is
// frozen: its theta is no longer updated, the lockstep sweeps it still takes part in do not change any of
// its outputs, and its `iterations` is the count at the freeze.  The final E-step runs once for both.
#pragma once
#include "pm_em_smem.cuh"

namespace pm {
namespace k {

constexpr int kPairMaxWarps = 10;  // 12 was measured no faster and caps the kernel at 80 registers
constexpr int kPairMaxSeqs = 64;     // small sets: per-sequence state (previous maxima, metadata) lives in shared memory;
                                     // large sets: at most this many sequences per tile
constexpr int kPairMaxWords = 2048;  // small sets: packed words of the whole set, staged once per CTA by one TMA bulk copy
// Two different l-mers whose FP64 weights (under this kernel's theta) lie closer than this go to the FP64 kernel.  The
// FP32 error of the M-step sums is ~1e-6 in a window weight.  EM amplifies an asymmetry eps between two equally good
// windows of one sequence: the cells they touch move by eps / count, the weight gap by up to 2 l eps / count, the
// responsibilities by a quarter of that -- a factor l / (2 count) per iteration, count being the column mass behind a
// cell, which grows with the number of sequences t.  The window widens as 50 / t, up to ten times: 5e-6 at t = 20 (every
// BASELINE configuration; the campaign found gaps of 1e-9 in the reference that this kernel saw as 2.7e-6 and 3.8e-6 at
// t = 21 and 16 -- a theta cell of 0.03 carries ~6e-8 of absolute error, 2e-6 relative, once per differing column),
// 2e-5 on sets of five sequences or fewer, where the amplification reaches ~l/2.  (A gap that EM has already blown up
// beyond the window cannot be seen from the final state.)
constexpr double kPairTieAbs = 2e-6, kPairTieRel = 1e-7, kPairTieAmpMax = 10.0;
constexpr int kPairNearCap = 64;     // near-maximum windows re-evaluated in FP64, per warp and bucket

// The per-sequence bookkeeping around the two hot loops is large straight-line code that every warp walks
// once per sequence; it is kept to ONE copy (rolled bucket loops, out-of-line FP64 exp/log) so the kernel
// stays inside the instruction cache.
__device__ __noinline__ double exp_f64(double x) { return exp(x); }
__device__ __noinline__ double log_f64(double x) { return log(x); }

__device__ __forceinline__ double window_weight_rolled(const double* __restrict__ D64, uint64_t v, int l) {
    double w0 = 0.0, w1 = 0.0;  // two chains: the sum is latency-bound
    int c = 0;
#pragma unroll 1
    for (; c + 1 < l; c += 2) {
        w0 += D64[c * 4 + (static_cast<unsigned>(v >> (62 - 2 * c)) & 3u)];
        w1 += D64[c * 4 + 4 + (static_cast<unsigned>(v >> (60 - 2 * c)) & 3u)];
    }
    if (c < l) w0 += D64[c * 4 + (static_cast<unsigned>(v >> (62 - 2 * c)) & 3u)];
    return w0 + w1;
}

// Packed FP32x2 arithmetic (sm_100: FADD2 / FMUL2 / FFMA2, one instruction for the two buckets of a pair; the
// results are the same round-to-nearest values as two scalar instructions).
__device__ __forceinline__ unsigned long long f2_pack(float2 v) {
    unsigned long long r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(v.x), "f"(v.y));
    return r;
}
__device__ __forceinline__ float2 f2_unpack(unsigned long long r) {
    float2 v;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(v.x), "=f"(v.y) : "l"(r));
    return v;
}
__device__ __forceinline__ float2 f2_add(float2 a, float2 b) {
    unsigned long long d;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(f2_pack(a)), "l"(f2_pack(b)));
    return f2_unpack(d);
}
__device__ __forceinline__ float2 f2_mul(float2 a, float2 b) {
    unsigned long long d;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(f2_pack(a)), "l"(f2_pack(b)));
    return f2_unpack(d);
}
__device__ __forceinline__ float2 f2_fma(float2 a, float2 b, float2 c) {
    unsigned long long d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(f2_pack(a)), "l"(f2_pack(b)), "l"(f2_pack(c)));
    return f2_unpack(d);
}

struct SeqAcc {
    float best_w, s_all, s_far;  // s_all doubles as the lane's second-best weight in the scouting final sweep
    int best_j, nnear, ncand;
    bool overflow;
};

// modes of pass A
constexpr int kPassFinal = 0;  // final sweep: stores w, tracks each lane's first maximum
constexpr int kPassExp = 1;    // EM sweep: stores e = exp(w - ref), sums, counts near candidates
constexpr int kPassScout = 2;  // final sweep without stores: each lane's first maximum and its second-best weight

__device__ __forceinline__ void near_push16(unsigned ball, bool keep, int lane, int j, uint16_t* __restrict__ my_near,
                                            int& nnear, bool& overflow) {
    if (ball && !overflow) {
        const int cnt = __popc(ball);
        if (nnear + cnt > kPairNearCap) {
            overflow = true;
        } else {
            if (keep) my_near[nnear + __popc(ball & ((1u << lane) - 1u))] = static_cast<uint16_t>(j);
            nnear += cnt;
        }
    }
}

// byte offset of pair-table entry (nibble g of the window) for 8-byte entries
template <int g>
__device__ __forceinline__ uint32_t nibble_off8(uint32_t vh, uint32_t vl) {
    return g < 7    ? (vh >> (25 - 4 * g)) & 0x78u
           : g == 7 ? (vh << 3) & 0x78u
           : g < 15 ? (vl >> (57 - 4 * g)) & 0x78u
                    : (vl << 3) & 0x78u;
}

template <int G, int g = 0>
struct PairLookup {
    static __device__ __forceinline__ void run(const float2* __restrict__ T2, uint32_t vh, uint32_t vl, float2* t) {
        t[g] = *reinterpret_cast<const float2*>(reinterpret_cast<const char*>(T2) + g * 128 + nibble_off8<g>(vh, vl));
        PairLookup<G, g + 1>::run(T2, vh, vl, t);
    }
    static __device__ __forceinline__ void run1(const float* __restrict__ Tb, uint32_t vh, uint32_t vl, float* t) {
        t[g] = *reinterpret_cast<const float*>(reinterpret_cast<const char*>(Tb) + g * 128 + nibble_off8<g>(vh, vl));
        PairLookup<G, g + 1>::run1(Tb, vh, vl, t);
    }
};
template <int G>
struct PairLookup<G, G> {
    static __device__ __forceinline__ void run(const float2*, uint32_t, uint32_t, float2*) {}
    static __device__ __forceinline__ void run1(const float*, uint32_t, uint32_t, float*) {}
};

// log-odds of one window under both buckets' pair tables (FP32, pairwise-tree sums)
template <int G>
__device__ __forceinline__ void pair_weights(const float2* __restrict__ T2, uint32_t vh, uint32_t vl, float& w0, float& w1) {
    float2 t[G];
    PairLookup<G>::run(T2, vh, vl, t);
#pragma unroll
    for (int s = 1; s < G; s <<= 1) {
#pragma unroll
        for (int g = 0; g + s < G; g += 2 * s) t[g] = f2_add(t[g], t[g + s]);
    }
    w0 = t[0].x;
    w1 = t[0].y;
}

// one bucket only (Tb = the float view of T2 offset by the bucket): same association as pair_weights
template <int G>
__device__ __forceinline__ float single_weight(const float* __restrict__ Tb, uint32_t vh, uint32_t vl) {
    float t[G];
    PairLookup<G>::run1(Tb, vh, vl, t);
#pragma unroll
    for (int s = 1; s < G; s <<= 1) {
#pragma unroll
        for (int g = 0; g + s < G; g += 2 * s) t[g] += t[g + s];
    }
    return t[0];
}

template <int kMode, bool kTail>
__device__ __forceinline__ void pair_finish(float w0, float w1, int j, bool live, float2* __restrict__ zq, float ref2a,
                                            float ref2b, float near_thr, SeqAcc& a, SeqAcc& b);

// one 32-window chunk of pass A in the given mode (see kPassFinal / kPassExp / kPassScout)
template <int G, int kMode, bool kTail>
__device__ __forceinline__ void pair_chunk(const float2* __restrict__ T2, uint32_t vh, uint32_t vl, int j, bool live,
                                           float2* __restrict__ zq, float ref2a, float ref2b, float near_thr, SeqAcc& a,
                                           SeqAcc& b) {
    float w0 = -INFINITY, w1 = -INFINITY;
    if (!kTail || live) pair_weights<G>(T2, vh, vl, w0, w1);
    pair_finish<kMode, kTail>(w0, w1, j, live, zq, ref2a, ref2b, near_thr, a, b);
}

// second half of pair_chunk: from the two weights to the stored value and the running sums
template <int kMode, bool kTail>
__device__ __forceinline__ void pair_finish(float w0, float w1, int j, bool live, float2* __restrict__ zq, float ref2a,
                                            float ref2b, float near_thr, SeqAcc& a, SeqAcc& b) {
    if (!kTail || live) {
        if (kMode == kPassExp) {
            const float2 arg = f2_fma(make_float2(w0, w1), make_float2(kLog2e, kLog2e), make_float2(-ref2a, -ref2b));
            const float e0 = fast_ex2(arg.x);
            const float e1 = fast_ex2(arg.y);
            *zq = make_float2(e0, e1);
            a.s_all += e0;
            b.s_all += e1;
            a.ncand += e0 >= near_thr ? 1 : 0;
            b.ncand += e1 >= near_thr ? 1 : 0;
        } else if (kMode == kPassFinal) {
            *zq = make_float2(w0, w1);
        }
    }
    if (kMode == kPassExp) {
        a.best_w = fmaxf(a.best_w, w0);
        b.best_w = fmaxf(b.best_w, w1);
    } else {
        if (kMode == kPassScout) {  // second-best weight seen by this lane (-inf for dead tail lanes)
            a.s_all = fmaxf(a.s_all, fminf(w0, a.best_w));
            b.s_all = fmaxf(b.s_all, fminf(w1, b.best_w));
        }
        if (w0 > a.best_w) {  // strict: the earliest offset is kept
            a.best_w = w0;
            a.best_j = j;
        }
        if (w1 > b.best_w) {
            b.best_w = w1;
            b.best_j = j;
        }
    }
}

template <int G, int kMode>
__device__ __forceinline__ void pair_pass_a(const float2* __restrict__ T2, const uint64_t* __restrict__ wp, int W, int lane,
                                            float2* __restrict__ zs, float refa, float refb, float near_thr, SeqAcc& a,
                                            SeqAcc& b) {
    const float ref2a = refa * kLog2e, ref2b = refb * kLog2e;
    uint64_t hi = wp[0];
    const uint64_t* __restrict__ wq = wp + 1;
    float2* __restrict__ zq = zs + lane;
    int j = lane;
    // two chunks per trip: all sixteen table lookups are issued before the first dependent add (the compiler
    // does not move shared-memory loads across the z stores on its own)
    for (const int j_two = (W & ~63); j < j_two; j += 64) {
        const uint64_t lo1 = wq[0], lo2 = wq[1];
        wq += 2;
        uint32_t vh1, vl1, vh2, vl2;
        window_halves(hi, lo1, lane, vh1, vl1);
        window_halves(lo1, lo2, lane, vh2, vl2);
        hi = lo2;
        float w0, w1, w2, w3;
        pair_weights<G>(T2, vh1, vl1, w0, w1);
        pair_weights<G>(T2, vh2, vl2, w2, w3);
        pair_finish<kMode, false>(w0, w1, j, true, zq, ref2a, ref2b, near_thr, a, b);
        pair_finish<kMode, false>(w2, w3, j + 32, true, zq + 32, ref2a, ref2b, near_thr, a, b);
        zq += 64;
    }
    for (const int j_full = W & ~31; j < j_full; j += 32) {
        const uint64_t lo = *wq++;
        uint32_t vh, vl;
        window_halves(hi, lo, lane, vh, vl);
        hi = lo;
        pair_chunk<G, kMode, false>(T2, vh, vl, j, true, zq, ref2a, ref2b, near_thr, a, b);
        zq += 32;
    }
    if ((W & 31) != 0) {
        uint32_t vh, vl;
        window_halves(hi, *wq, lane, vh, vl);
        pair_chunk<G, kMode, true>(T2, vh, vl, j, j < W, zq, ref2a, ref2b, near_thr, a, b);
    }
}

// one bucket, plain weights into its half of the interleaved buffer (fallback when the maximum moved too far)
template <int G>
__device__ __forceinline__ void single_pass_w(const float* __restrict__ Tb, const uint64_t* __restrict__ wp, int W, int lane,
                                              float* __restrict__ zb, float& best_w) {
    const int chunks = (W + 31) >> 5;
    uint64_t hi = wp[0];
    for (int c = 0; c < chunks; ++c) {
        const uint64_t lo = wp[c + 1];
        uint32_t vh, vl;
        window_halves(hi, lo, lane, vh, vl);
        hi = lo;
        const int j = (c << 5) + lane;
        if (j < W) {
            const float w = single_weight<G>(Tb, vh, vl);
            zb[2 * j] = w;
            best_w = fmaxf(best_w, w);
        }
    }
}

// sweep over one bucket's stored values (stride 2): kFromW turns stored w into e = exp(w - M) first
template <bool kFromW>
__device__ __forceinline__ void pair_detect(float* __restrict__ zb, int W, int lane, float M, float thr, float& s_all,
                                            float& s_far, uint16_t* __restrict__ my_near, int& nnear, bool& overflow) {
    const int chunks = (W + 31) >> 5;
    for (int c = 0; c < chunks; ++c) {
        const int j = (c << 5) + lane;
        float e = 0.f;
        bool keep = false;
        if (j < W) {
            e = zb[2 * j];
            if (kFromW) {
                e = fast_ex2((e - M) * kLog2e);
                zb[2 * j] = e;
            }
            keep = e >= thr;
        }
        s_all += e;
        s_far += keep ? 0.f : e;
        near_push16(__ballot_sync(0xffffffffu, keep), keep, lane, j, my_near, nnear, overflow);
    }
}

// pair_detect<false> for both buckets in one sweep over the interleaved values (a bucket whose flag is off is
// left untouched)
__device__ __forceinline__ void pair_detect_both(const float2* __restrict__ zs, int W, int lane, bool on_a, bool on_b,
                                                 float thr_a, float thr_b, SeqAcc& a, SeqAcc& b,
                                                 uint16_t* __restrict__ near_a, uint16_t* __restrict__ near_b) {
    float far_a = 0.f, far_b = 0.f;
    int n_a = 0, n_b = 0;
    bool ov_a = !on_a, ov_b = !on_b;  // an overflowed list takes no more entries
    const int chunks = (W + 31) >> 5;
    for (int c = 0; c < chunks; ++c) {
        const int j = (c << 5) + lane;
        float2 e = make_float2(0.f, 0.f);
        if (j < W) e = zs[j];
        const bool k_a = j < W && e.x >= thr_a, k_b = j < W && e.y >= thr_b;
        far_a += k_a ? 0.f : e.x;
        far_b += k_b ? 0.f : e.y;
        near_push16(__ballot_sync(0xffffffffu, k_a), k_a, lane, j, near_a, n_a, ov_a);
        near_push16(__ballot_sync(0xffffffffu, k_b), k_b, lane, j, near_b, n_b, ov_b);
    }
    if (on_a) a.s_far = far_a, a.nnear = n_a, a.overflow = ov_a;
    if (on_b) b.s_far = far_b, b.nnear = n_b, b.overflow = ov_b;
}

// After pass A of one sequence, one bucket: settle the reference maximum, the near list and the normaliser.
// Returns 1/total; ref is updated when the fallback re-based the stored values on M.  The near list (windows
// with e >= near_e, i.e. within log_z_eps of the maximum) is built by a second light sweep over the stored
// values, and only when it can be short enough to be used: pass A merely counted the candidates against a
// threshold kNearMargin below the previous maximum.
template <int G>
__device__ __forceinline__ float pair_settle(const float* __restrict__ Tb, const uint64_t* __restrict__ wp, int W, int lane,
                                             float* __restrict__ zb, uint16_t* __restrict__ my_near, SeqAcc& a, float& ref,
                                             float& M, float total, int n_cand, float& near_e, float log_z_eps,
                                             bool force_rebuild, bool want_near, int* bad) {
    // M (in/out), total and n_cand are the warp-wide max / sum / count of pass A, reduced by the caller for both
    // buckets at once
    constexpr float kNearMargin = 4.f;
    if (!(M > -INFINITY) || !(M < INFINITY)) *bad = 1;
    const float shift = M - ref;
    const bool have_e = shift > -60.f && shift < 60.f && total > 0.f && total < INFINITY;
    if (!have_e) {
        // the maximum is too far from the reference for FP32 range: redo this bucket as two passes
        __syncwarp();
        float bw = -INFINITY;
        single_pass_w<G>(Tb, wp, W, lane, zb, bw);
        M = warp_max_f(bw);
        if (!(M > -INFINITY) || !(M < INFINITY)) *bad = 1;
        __syncwarp();
        ref = M;
        near_e = fast_ex2(log_z_eps * kLog2e);
        a.s_all = 0.f, a.s_far = 0.f, a.nnear = 0, a.overflow = false;
        pair_detect<true>(zb, W, lane, M, near_e, a.s_all, a.s_far, my_near, a.nnear, a.overflow);
        total = warp_sum_f(a.s_all);
    } else {
        near_e = fast_ex2((shift + log_z_eps) * kLog2e);
        a.overflow = true;
        if (want_near) {
            // the count is an upper bound of the list length unless the maximum dropped below the margin
            // the sweep that builds the list is left to the caller, who runs it once for both buckets
            if (force_rebuild || M < ref - kNearMargin || n_cand <= kPairNearCap) a.nnear = -2;
        }
    }
    if (!(total > 0.f)) *bad = 1;
    return 1.f / total;
}

// transposed warp reduction of N values (N = 16 or 32): afterwards lane L holds the warp-wide sum of
// v[(L * N) >> 5] in v[0] (both lanes of a pair for N = 16)
template <int N>
__device__ __forceinline__ float warp_transpose_sum(float (&v)[N], int lane) {
#pragma unroll
    for (int n = N / 2, o = 16; n >= 1; n >>= 1, o >>= 1) {
        const bool up = (lane & o) != 0;
#pragma unroll
        for (int i = 0; i < n; ++i) {
            const float keep = up ? v[i + n] : v[i];
            const float send = up ? v[i] : v[i + n];
            v[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
        }
    }
    if (N == 16) v[0] += __shfl_xor_sync(0xffffffffu, v[0], 1);
    return v[0];
}

template <int G>
__global__ void __launch_bounds__(kPairMaxWarps * 32, 2)
em_refine_pair_kernel(const EmParams p, const EmSmemExtra x) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int nwarps = blockDim.x >> 5;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int l = p.l, t = p.t;
    const int TH = 4 * (l + 1);
    // Small sets (every t=20 configuration): metadata and previous maxima of all sequences in shared memory, the
    // whole packed set staged once.  Large sets: the same kernel walks the tiles with the metadata of the
    // current tile only, the previous maxima in a per-CTA global scratch and the packed words of each tile
    // double-buffered by TMA (the next tile's words arrive while the current tile is processed).
    const bool big = x.mprev_g != nullptr;
    const int tpad = big ? kPairMaxSeqs : ((t + 1) & ~1);
    constexpr int NV = 2 * G <= 16 ? 16 : 32;  // values per class flush (2 buckets x G column pairs, padded)

    // ---- shared memory carve-up (mirrored by em_pair_smem_bytes on the host)
    double* thd = reinterpret_cast<double*>(smem_raw);        // [2][TH] theta, cell 4c+r, column 0 = background
    double* D64 = thd + 2 * TH;                               // [2][TH] log theta[r][c+1] - log theta[r][0]
    double* L64 = D64 + 2 * TH;                               // [2][TH] log max(theta, 1e-9), written with theta
    double* llpart = L64 + 2 * TH;                            // [nwarps][2]
    double* dscal = llpart + 2 * nwarps;                      // [2][6]: [0] previous LL, [2..5] log background
    float2* T2 = reinterpret_cast<float2*>(dscal + 12);       // [G][16] {bucket 0, bucket 1}
    float* Cq = reinterpret_cast<float*>(T2 + 16 * G);        // [2][16][G] class sums
    float* cpart = Cq + 32 * G;                               // [16 + nwarps][NV] slot = warp + class
    float* mprev_s = cpart + (16 + nwarps) * NV;              // [2][tpad] previous per-sequence maxima (small sets)
    float* ubs = mprev_s + 2 * tpad;                          // [2] upper bound of any window weight (+2 pad)
    int* prof = reinterpret_cast<int*>(ubs + 4);              // [2][128]
    int* iscal = prof + 256;                                  // [2][4]: [0] stop [1] score [2] bad [3] iterations
    int* s_off = iscal + 8;                                   // [17] first row of each class (+3 pad)
    int* wrow = s_off + 20;                                   // [nwarps + 1] class-row range of each warp (16 slots)
    int* smeta = wrow + 16;                                  // [tpad][4]: word offset, windows, z offset, z slots
    unsigned long long* cons_bits = reinterpret_cast<unsigned long long*>(smeta + 4 * tpad);  // [2]
    uint16_t* near_j = reinterpret_cast<uint16_t*>(cons_bits + 2);                            // [nwarps][2][kPairNearCap]
    // offsets are aligned as integers (smem_raw is 16-byte aligned) so that every pointer below stays a
    // provable shared-memory address: LDS/STS, not generic loads
    const unsigned int z_off = (static_cast<unsigned int>(reinterpret_cast<unsigned char*>(near_j + nwarps * 2 * kPairNearCap) - smem_raw) + 15u) & ~15u;
    float2* zbuf = reinterpret_cast<float2*>(smem_raw + z_off);
    uint64_t* wstage = reinterpret_cast<uint64_t*>(smem_raw + z_off + static_cast<unsigned int>((x.zcap + 1) & ~1) * 8u);
    unsigned long long* mbar = reinterpret_cast<unsigned long long*>(wstage + static_cast<size_t>(x.wcap) * (big ? 2 : 1));
    float* mprev = big ? x.mprev_g + static_cast<size_t>(blockIdx.x) * 2 * t : mprev_s;
    const int mstride = big ? t : tpad;  // bucket 1's maxima follow bucket 0's
    unsigned int visit = 0;              // tiles visited (large sets): stage = visit & 1, parity = (visit >> 1) & 1

    // ---- packed words of the whole set: one TMA bulk copy per CTA, resident for every bucket
    const int64_t word0 = x.tiles[0].word_begin;
    if (threadIdx.x == 0) {
        mbar_init(&mbar[0], 1);
        mbar_init(&mbar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        // small sets: the whole set; large sets: the first tile (wcap = the largest tile)
        const unsigned bytes = static_cast<unsigned>(big ? x.tiles[0].n_words : x.wcap) * 8u;
        mbar_expect_tx(&mbar[0], bytes);
        tma_load_1d(wstage, p.words + word0, bytes, &mbar[0]);
    }
    if (!big) {
        for (int i = threadIdx.x; i < t; i += blockDim.x) {
            smeta[4 * i + 0] = static_cast<int>(p.word_off[i] - word0);
            smeta[4 * i + 1] = p.seq_len[i] - l + 1;
            smeta[4 * i + 2] = x.seq_zoff[i];
            smeta[4 * i + 3] = static_cast<int>(p.win_off[i]);  // first flat l-mer index of the sequence
        }
    }
    // Slots that are not window starts (front pad, the last l-1 bases of a sequence, balancing gaps) must read as
    // zero in the M-step gather and are never written by a sweep.  With a single tile the layout never changes:
    // zero the buffer once; with several tiles the buffer is re-laid out per tile and those slots are re-zeroed.
    const bool rezero = x.n_tiles > 1;
    for (int k = threadIdx.x; k < x.zcap; k += blockDim.x) zbuf[k] = make_float2(0.f, 0.f);
    // sum_i log W_i, used by the two threads that close an iteration: block-wide sum, fixed order
    double sum_logw = 0.0;
    {
        double part = 0.0;
        for (int i = threadIdx.x; i < t; i += blockDim.x) part += p.seq_logw[i];
        part = warp_sum_d(part);
        if (lane == 0) llpart[warp] = part;
    }
    __syncthreads();
    for (int w = 0; w < nwarps; ++w) sum_logw += llpart[w];
    if (!big) mbar_wait(&mbar[0], 0);
    __syncthreads();  // llpart is reused by the iterations
    uint16_t* near_a = near_j + (warp * 2 + 0) * kPairNearCap;
    uint16_t* near_b = near_j + (warp * 2 + 1) * kPairNearCap;
    const int colshift = 62 - 2 * lane;
    const float* T2f = reinterpret_cast<const float*>(T2);
    float* zf = reinterpret_cast<float*>(zbuf);

    const unsigned int n_work = p.n_work_dev ? *p.n_work_dev : p.n_work;
    const unsigned int n_pairs = (n_work + 1) >> 1;
    for (unsigned int pi = blockIdx.x; pi < n_pairs; pi += gridDim.x) {
        const bool live1 = 2 * pi + 1 < n_work;
        const unsigned int wis[2] = {2 * pi, live1 ? 2 * pi + 1 : 2 * pi};  // an odd tail refines its bucket twice
        const WorkDesc wd0 = p.work[wis[0]], wd1 = p.work[wis[1]];
        // output slots: the work index itself, or its slot in the list the work items were compacted from
        const unsigned int ois[2] = {p.out_map ? p.out_map[wis[0]] : wis[0], p.out_map ? p.out_map[wis[1]] : wis[1]};
        __syncthreads();
#ifdef PM_EM_TIMING
        long long t_phase = clock64();
#endif

        // ---- init_model (refine.hpp:90-127), pseudocount 0
        #pragma unroll 1
        for (int i = threadIdx.x; i < 256; i += blockDim.x) prof[i] = 0;
        if (threadIdx.x < 2) {
            iscal[threadIdx.x * 4 + 0] = 0;
            iscal[threadIdx.x * 4 + 2] = 0;
            iscal[threadIdx.x * 4 + 3] = 0;
            dscal[threadIdx.x * 6] = 0.0;
        }
        __syncthreads();
        #pragma unroll 1
        for (unsigned int m = threadIdx.x; m < wd0.count + wd1.count; m += blockDim.x) {
            const int b = m >= wd0.count;
            const int64_t f = b ? p.members[wd1.mem_begin + (m - wd0.count)] : p.members[wd0.mem_begin + m];
            uint64_t v;
            if (!big) {
                int i = 0;
                for (int hi = t; hi - i > 1;) {  // owner of flat l-mer index f: largest i with win_off[i] <= f
                    const int mid = (i + hi) >> 1;
                    if (smeta[4 * mid + 3] <= f) i = mid; else hi = mid;
                }
                v = load_window(wstage + smeta[4 * i], f - smeta[4 * i + 3]);
            } else {
                const int i = seq_of_flat(p.win_off, t, f);
                v = load_window(p.words + p.word_off[i], f - p.win_off[i]);
            }
            #pragma unroll 1
            for (int c = 0; c < l; ++c) atomicAdd(&prof[b * 128 + c * 4 + (static_cast<unsigned>(v >> (62 - 2 * c)) & 3u)], 1);
        }
        __syncthreads();
        #pragma unroll 1
        for (int e2 = threadIdx.x; e2 < 2 * TH; e2 += blockDim.x) {
            const int b = e2 >= TH, e = e2 - b * TH;
            const int c = e >> 2, r = e & 3;
            // pm_em_step starts from a caller-supplied model instead of theta0
            const double tv = p.theta_in ? p.theta_in[static_cast<int64_t>(wis[b]) * TH + r * (l + 1) + c]
                              : c == 0   ? p.tot_sym[r] / p.tot_bases
                                         : static_cast<double>(prof[b * 128 + (c - 1) * 4 + r]) / static_cast<double>(b ? wd1.count : wd0.count);
            thd[e2] = tv;
            L64[e2] = log_f64(fmax(tv, 1e-9));
        }
        __syncthreads();

        PM_PHASE(0);  // init_model
        int iterations = 0;  // lockstep sweeps done
        bool stop0 = false, stop1 = false;
        bool final_pass = false;
        for (;;) {
            // ---- log tables of the current thetas (refine.hpp:155-161) from L64 = log max(theta, 1e-9), which the
            // thread that wrote a theta cell stored next to it: FP64 differences, rounded once to FP32
            #pragma unroll 1
            for (int e2 = threadIdx.x; e2 < 2 * 4 * l; e2 += blockDim.x) {
                const int b = e2 >= 4 * l, e = e2 - b * 4 * l;
                D64[b * TH + e] = L64[b * TH + e + 4] - L64[b * TH + (e & 3)];
            }
            if (threadIdx.x >= blockDim.x - 8) {
                const int k8 = threadIdx.x - (blockDim.x - 8);
                dscal[(k8 >> 2) * 6 + 2 + (k8 & 3)] = L64[(k8 >> 2) * TH + (k8 & 3)];
            }
            if (final_pass) {
                #pragma unroll 1
                for (int i = threadIdx.x; i < 256; i += blockDim.x) prof[i] = 0;
                if (threadIdx.x < 2) {
                    iscal[threadIdx.x * 4 + 1] = 0;
                    cons_bits[threadIdx.x] = 0ULL;
                }
            }
            #pragma unroll 1
            for (int e2 = threadIdx.x; e2 < 32 * G; e2 += blockDim.x) {
                const int b = e2 & 1, e = e2 >> 1;
                const int g = e >> 4, q = e & 15;
                const int c0 = 2 * g, c1 = 2 * g + 1;
                const double* L = L64 + b * TH;
                double v = 0.0;
                if (c0 < l) v = L[(c0 + 1) * 4 + (q >> 2)] - L[q >> 2];
                if (c1 < l) v += L[(c1 + 1) * 4 + (q & 3)] - L[q & 3];
                reinterpret_cast<float*>(T2)[e2] = static_cast<float>(v);
            }
            if (iterations == 0 && !final_pass && warp >= nwarps - 2) {
                // No window weight exceeds ub = the sum of the column maxima.  Iteration 0 takes its exponentials
                // relative to ub - 40: e <= exp(40) cannot overflow, and a sequence whose best window lies up to 100
                // below ub (four floored columns of theta0) still has its maximum inside the +-60 window that the
                // fused pass needs (at ub itself 47 % of the C1 sequences fell back to the two-pass form).
                const int b = warp - (nwarps - 2);
                const double* L = L64 + b * TH;
                const int c = lane + 1;
                double m = 0.0;
                if (lane < l) m = fmax(fmax(L[c * 4] - L[0], L[c * 4 + 1] - L[1]), fmax(L[c * 4 + 2] - L[2], L[c * 4 + 3] - L[3]));
                m = warp_sum_d(m);
                if (lane == 0) ubs[b] = static_cast<float>(m) - 40.f;
            }
            #pragma unroll 1
            for (int e = threadIdx.x; e < 32 * G; e += blockDim.x) Cq[e] = 0.f;
            __syncthreads();
            PM_PHASE(1);  // log tables

            double ll0 = 0.0, ll1 = 0.0;
            for (int tile_i = 0; tile_i < x.n_tiles; ++tile_i) {
                const TileDesc tile = x.tiles[tile_i];
                if (threadIdx.x < 17) s_off[threadIdx.x] = x.tile_group_off[tile_i * 17 + threadIdx.x];
                if (threadIdx.x >= 32 && threadIdx.x <= 32 + nwarps) {  // class rows [wrow[w], wrow[w+1]) belong to warp w
                    const int w = threadIdx.x - 32;
                    wrow[w] = static_cast<int>(static_cast<long long>(x.tile_group_off[tile_i * 17 + 16]) * w / nwarps);
                }
                const int sbase = big ? tile.seq_begin : 0;  // smeta holds sequence i at row i - sbase
                const uint64_t* __restrict__ wtile = wstage;
                if (big) {
                    for (int k = threadIdx.x; k < tile.seq_end - tile.seq_begin; k += blockDim.x) {
                        const int i = tile.seq_begin + k;
                        smeta[4 * k + 0] = static_cast<int>(p.word_off[i] - tile.word_begin);
                        smeta[4 * k + 1] = p.seq_len[i] - l + 1;
                        smeta[4 * k + 2] = x.seq_zoff[i];
                    }
                    if (x.n_tiles > 1) {
                        wtile = wstage + static_cast<size_t>(x.wcap) * (visit & 1);
                        if (threadIdx.x == 0) {  // prefetch the next tile of the cyclic walk into the other stage
                            const TileDesc nt = x.tiles[tile_i + 1 < x.n_tiles ? tile_i + 1 : 0];
                            unsigned long long* nb = &mbar[(visit + 1) & 1];
                            mbar_expect_tx(nb, static_cast<unsigned>(nt.n_words) * 8u);
                            tma_load_1d(wstage + static_cast<size_t>(x.wcap) * ((visit + 1) & 1), p.words + nt.word_begin,
                                        static_cast<unsigned>(nt.n_words) * 8u, nb);
                        }
                        mbar_wait(&mbar[visit & 1], (visit >> 1) & 1);
                        ++visit;
                    } else if (visit == 0) {
                        mbar_wait(&mbar[0], 0);
                        ++visit;
                    }
                    __syncthreads();  // metadata of the tile visible to every warp
                }
                if (rezero) {  // front pad (dummy lanes of the class rows read it)
                    for (int k = threadIdx.x, k_end = smeta[4 * (tile.seq_begin - sbase) + 2]; k < k_end; k += blockDim.x)
                        zbuf[k] = make_float2(0.f, 0.f);
                }
                // ================= E-step: warp per sequence of the tile =================
                for (int i = tile.seq_begin + warp; i < tile.seq_end; i += nwarps) {
                    const int si = i - sbase;
                    const uint64_t* __restrict__ wp = wtile + smeta[4 * si];
                    const int W = smeta[4 * si + 1];
                    const int zo = smeta[4 * si + 2];
                    const int chunks = (W + 31) >> 5;
                    float2* zs = zbuf + zo;
                    float* zb0 = zf + 2 * zo;
                    if (rezero) {
                        // slots that are not window starts read as zero in the M-step gather
                        const int z_end = (i + 1 < tile.seq_end ? smeta[4 * (si + 1) + 2] : tile.zlen) - zo;
                        #pragma unroll 1
                        for (int k = W + lane; k < z_end; k += 32) zs[k] = make_float2(0.f, 0.f);
                    }
                    SeqAcc a = {-INFINITY, 0.f, 0.f, 0, 0, 0, false}, b = {-INFINITY, 0.f, 0.f, 0, 0, 0, false};

                    if (final_pass) {
                        // ---- positions: per-sequence argmax, ties to the smallest offset (refine.hpp:311-316).
                        // Windows within delta of the FP32 maximum are compared by their FP64 weights.  A scouting
                        // sweep without stores settles the common case of a single window within delta (it IS the
                        // argmax); only sequences with near-ties take the storing sweep and the FP64 comparison.
                        a.s_all = -INFINITY, b.s_all = -INFINITY;
                        pair_pass_a<G, kPassScout>(T2, wp, W, lane, zs, 0.f, 0.f, 0.f, a, b);
                        const float Mf0 = warp_max_f(a.best_w), Mf1 = warp_max_f(b.best_w);
                        if (!(Mf0 > -INFINITY) || !(Mf0 < INFINITY)) iscal[2] = 1;
                        if (!(Mf1 > -INFINITY) || !(Mf1 < INFINITY)) iscal[6] = 1;
                        float lim0 = Mf0 - (1e-3f + 1e-5f * fabsf(Mf0)), lim1 = Mf1 - (1e-3f + 1e-5f * fabsf(Mf1));
                        const unsigned near0 = __ballot_sync(0xffffffffu, a.best_w >= lim0), near1 = __ballot_sync(0xffffffffu, b.best_w >= lim1);
                        const bool uniq0 = __popc(near0) == 1 && !__any_sync(0xffffffffu, a.s_all >= lim0);
                        const bool uniq1 = __popc(near1) == 1 && !__any_sync(0xffffffffu, b.s_all >= lim1);
                        if (uniq0) {  // as if the list held exactly this window
                            a.nnear = -1;
                            a.best_j = __shfl_sync(0xffffffffu, a.best_j, __ffs(near0) - 1);
                        }
                        if (uniq1) {
                            b.nnear = -1;
                            b.best_j = __shfl_sync(0xffffffffu, b.best_j, __ffs(near1) - 1);
                        }
                        if (!(uniq0 && uniq1)) {
                            const int keep_j0 = a.best_j, keep_j1 = b.best_j;
                            a.best_w = -INFINITY, b.best_w = -INFINITY;
                            pair_pass_a<G, kPassFinal>(T2, wp, W, lane, zs, 0.f, 0.f, 0.f, a, b);
                            __syncwarp();
                            if (uniq0) a.best_j = keep_j0;
                            if (uniq1) b.best_j = keep_j1;
                            if (uniq0) lim0 = INFINITY;  // already settled: list nothing
                            if (uniq1) lim1 = INFINITY;
                            for (int c = 0; c < chunks; ++c) {
                                const int j = (c << 5) + lane;
                                bool k0 = false, k1 = false;
                                if (j < W) {
                                    const float2 w2 = zs[j];
                                    k0 = w2.x >= lim0;
                                    k1 = w2.y >= lim1;
                                }
                                near_push16(__ballot_sync(0xffffffffu, k0), k0, lane, j, near_a, a.nnear, a.overflow);
                                near_push16(__ballot_sync(0xffffffffu, k1), k1, lane, j, near_b, b.nnear, b.overflow);
                            }
                        }
                        __syncwarp();
#pragma unroll 1
                        for (int bb = 0; bb < 2; ++bb) {
                            const SeqAcc s = bb ? b : a;
                            const uint16_t* my_near = near_a + bb * kPairNearCap;
                            int arg;
                            if (s.nnear < 0) {
                                arg = s.best_j;  // the only window within delta of the maximum
                            } else if (!s.overflow) {
                                const double* D = D64 + bb * TH;
                                double bw = -INFINITY, sw = -INFINITY;  // best and runner-up weight, with their windows
                                int bj = 0x7fffffff, sj = 0x7fffffff;
                                auto offer = [&](double w, int j) {
                                    if (w > bw || (w == bw && j < bj)) {
                                        sw = bw;
                                        sj = bj;
                                        bw = w;
                                        bj = j;
                                    } else if (w > sw || (w == sw && j < sj)) {
                                        sw = w;
                                        sj = j;
                                    }
                                };
                                for (int e = lane; e < s.nnear; e += 32) {
                                    const int j = my_near[e];
                                    offer(window_weight_rolled(D, load_window(wp, j), l), j);
                                }
#pragma unroll
                                for (int o = 16; o > 0; o >>= 1) {
                                    const double ow = __shfl_xor_sync(0xffffffffu, bw, o), osw = __shfl_xor_sync(0xffffffffu, sw, o);
                                    const int oj = __shfl_xor_sync(0xffffffffu, bj, o), osj = __shfl_xor_sync(0xffffffffu, sj, o);
                                    offer(ow, oj);
                                    offer(osw, osj);
                                }
                                arg = bj;
                                // Two DIFFERENT l-mers whose weights lie closer than this kernel's theta can tell apart: the
                                // comparison above is exact for the theta at hand, but theta carries the FP32 error of the
                                // M-step sums (measured |d theta| <= 3.4e-7; typically ~1e-6 in a window weight), so which
                                // window wins in the reference (refine.hpp:165-186, :311-316) is decided by the FP64 kernel.
                                // (The same l-mer twice has bit-identical weights everywhere: the smaller offset wins, as
                                // above.)  Not for large sets: an FP64 refinement of 10^7 windows takes seconds per bucket.
                                // The runner-up that matters is the best window showing ANOTHER l-mer: repeats of the winning
                                // l-mer (homopolymer runs, tandem copies) tie exactly and must not hide it.
                                if (!big && p.flag_exact != nullptr && (bb == 0 || live1) && sj != 0x7fffffff) {
                                    const uint64_t bv = load_window(wp, bj) >> (64 - 2 * l);
                                    double dw = -INFINITY;
                                    for (int e = lane; e < s.nnear; e += 32) {
                                        const uint64_t v = load_window(wp, my_near[e]);
                                        if ((v >> (64 - 2 * l)) != bv) dw = fmax(dw, window_weight_rolled(D, v, l));
                                    }
#pragma unroll
                                    for (int o = 16; o > 0; o >>= 1) dw = fmax(dw, __shfl_xor_sync(0xffffffffu, dw, o));
                                    // count ~ t: the window is 5e-6 at t = 20, the FP32 one (2e-6) from t = 50 on and ten times that for t <= 5
                                    const double amp = fmin(kPairTieAmpMax, fmax(1.0, 50.0 / static_cast<double>(t)));
                                    if (lane == 0 && bw - dw <= amp * (kPairTieAbs + kPairTieRel * fabs(bw))) p.flag_exact[ois[bb]] = 1;
                                }
                            } else {
                                float bw = s.best_w;
                                int bj = s.best_j;
#pragma unroll
                                for (int o = 16; o > 0; o >>= 1) {
                                    const float ow = __shfl_xor_sync(0xffffffffu, bw, o);
                                    const int oj = __shfl_xor_sync(0xffffffffu, bj, o);
                                    if (ow > bw || (ow == bw && oj < bj)) {
                                        bw = ow;
                                        bj = oj;
                                    }
                                }
                                arg = bj;
                                // more near-maximum windows than the list holds: FP32 cannot order them
                                if (!big && p.flag_exact != nullptr && lane == 0 && (bb == 0 || live1)) p.flag_exact[ois[bb]] = 1;
                            }
                            if (p.out_pos && lane == 0 && (bb == 0 || live1)) p.out_pos[static_cast<int64_t>(ois[bb]) * t + i] = arg + 1;
                            if (lane < l) {
                                const uint64_t v = load_window(wp, arg);
                                atomicAdd(&prof[bb * 128 + lane * 4 + (static_cast<unsigned>(v >> colshift) & 3u)], 1);
                            }
                            __syncwarp();
                        }
                        continue;
                    }

                    // pass A with the exp fused in, taken relative to the previous iteration's maximum of this
                    // sequence (iteration 0: the upper bound); softmax is shift-invariant
                    constexpr float kNearMargin = 4.f;
                    const bool first = iterations == 0;
                    float ref0 = first ? ubs[0] : mprev[i];
                    float ref1 = first ? ubs[1] : mprev[mstride + i];
                    // iteration 0 lists nothing on the way (its reference is far above the maximum): rebuilt below
                    const float near_thr = first ? INFINITY : fast_ex2((p.log_z_eps - kNearMargin) * kLog2e);
                    pair_pass_a<G, kPassExp>(T2, wp, W, lane, zs, ref0, ref1, near_thr, a, b);
                    float M0 = 0.f, M1 = 0.f, inv0 = 0.f, inv1 = 0.f, ne0 = 0.f, ne1 = 0.f;
                    // the FP64 pass is skipped in the last iteration of the budget: its likelihood can no longer
                    // stop the loop (refine.hpp:296-304), so no near list is needed there
                    const bool want_near = iterations + 1 < p.max_iters;
                    // warp-wide max / sum / candidate count of both buckets, their shuffle chains interleaved
                    M0 = warp_max_f(a.best_w), M1 = warp_max_f(b.best_w);
                    float tot0 = a.s_all, tot1 = b.s_all;
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) {
                        tot0 += __shfl_xor_sync(0xffffffffu, tot0, o);
                        tot1 += __shfl_xor_sync(0xffffffffu, tot1, o);
                    }
                    const int nc0 = __reduce_add_sync(0xffffffffu, a.ncand), nc1 = __reduce_add_sync(0xffffffffu, b.ncand);
#pragma unroll 1
                    for (int bb = 0; bb < 2; ++bb) {  // rolled: one copy of the code for both buckets
                        SeqAcc s = bb ? b : a;
                        float ref = bb ? ref1 : ref0, M = bb ? M1 : M0, ne;
                        const float inv = pair_settle<G>(T2f + bb, wp, W, lane, zb0 + bb, near_a + bb * kPairNearCap, s, ref, M,
                                                         bb ? tot1 : tot0, bb ? nc1 : nc0, ne, p.log_z_eps, first, want_near,
                                                         &iscal[bb * 4 + 2]);
                        __syncwarp();  // every lane has read this sequence's previous maximum
                        if (lane == 0) mprev[bb * mstride + i] = M;
                        if (bb) {
                            b = s, ref1 = ref, M1 = M, inv1 = inv, ne1 = ne;
                        } else {
                            a = s, ref0 = ref, M0 = M, inv0 = inv, ne0 = ne;
                        }
                    }
                    __syncwarp();
                    if (a.nnear == -2 || b.nnear == -2) {
                        pair_detect_both(zs, W, lane, a.nnear == -2, b.nnear == -2, ne0, ne1, a, b, near_a, near_b);
                        __syncwarp();
                    }
                    // pass C: z_j = e_j / sum, both buckets
                    {
                        const float2 inv2 = make_float2(inv0, inv1);
                        int j = lane;
                        for (const int j4 = W - 96; j < j4; j += 128) {  // four chunks per trip: loads first, then stores
                            const float2 e0 = zs[j], e1 = zs[j + 32], e2 = zs[j + 64], e3 = zs[j + 96];
                            zs[j] = f2_mul(e0, inv2), zs[j + 32] = f2_mul(e1, inv2);
                            zs[j + 64] = f2_mul(e2, inv2), zs[j + 96] = f2_mul(e3, inv2);
                        }
                        for (; j < W; j += 32) zs[j] = f2_mul(zs[j], inv2);
                    }
                    __syncwarp();
                    // ---- log sum_j exp(w_j) per bucket; the FP32 form needs log(1/total): one logf for both buckets
                    // (odd lanes take bucket 1)
                    const float lg = logf((lane & 1) ? inv1 : inv0);
                    const float lg0 = __shfl_sync(0xffffffffu, lg, 0), lg1 = __shfl_sync(0xffffffffu, lg, 1);
#pragma unroll 1
                    for (int bb = 0; bb < 2; ++bb) {
                        const SeqAcc s = bb ? b : a;
                        float* zb = zb0 + bb;
                        const uint16_t* my_near = near_a + bb * kPairNearCap;
                        // the list holds exactly the windows with e >= near_e (lane L owns entries L and L + 32)
                        const bool n_a = !s.overflow && lane < s.nnear, n_b = !s.overflow && lane + 32 < s.nnear;
                        const float ref = bb ? ref1 : ref0, M = bb ? M1 : M0;
                        double lse;
                        if (!s.overflow) {
                            // FP64 re-evaluation of the dominant windows; the far tail (each < eps of the maximum)
                            // keeps its FP32 sum, rescaled from ref to M
                            const double* D = D64 + bb * TH;
                            const double far = static_cast<double>(warp_sum_f(s.s_far) * fast_ex2((ref - M) * kLog2e));
                            double wa = -INFINITY, wb = -INFINITY;
                            if (n_a) wa = window_weight_rolled(D, load_window(wp, my_near[lane]), l);
                            if (__any_sync(0xffffffffu, n_b)) {
                                if (n_b) wb = window_weight_rolled(D, load_window(wp, my_near[lane + 32]), l);
                            }
                            const double m64 = warp_max_d(fmax(wa, wb));
                            wa = n_a ? exp_f64(wa - m64) : 0.0;
                            if (__any_sync(0xffffffffu, n_b)) wb = n_b ? exp_f64(wb - m64) : 0.0; else wb = 0.0;
                            // far * exp(M - m64): |M - m64| ~ 1e-5 and far < W*eps, so first order is exact to ~1e-17
                            const double s64 = warp_sum_d(wa + wb) + far * (1.0 + (static_cast<double>(M) - m64));
                            lse = m64 + log_f64(s64);
                            if (n_a) zb[2 * my_near[lane]] = static_cast<float>(wa / s64);
                            if (n_b) zb[2 * my_near[lane + 32]] = static_cast<float>(wb / s64);
                        } else {
                            lse = static_cast<double>(ref) - static_cast<double>(bb ? lg1 : lg0);  // total is relative to ref
                        }
                        // log P(S_i) = log prod theta_bg - log W + logsumexp_j w_ij (refine.hpp:200); the first two
                        // terms are summed over the set by the thread that closes the iteration
                        if (bb) ll1 += lse; else ll0 += lse;
                    }
                    __syncwarp();
                }
                if (final_pass) {
                    if (tile_i + 1 < x.n_tiles) __syncthreads();  // the next tile reuses the z buffer
                    continue;
                }
                __syncthreads();
                PM_PHASE(2);  // E-step (warp 0's sequences + wait for the slowest warp)

                // ================= M-step of the tile: conflict-free class gather, both buckets =================
                {
                    const int item_lo = wrow[warp], item_hi = wrow[warp + 1];
                    // this warp's rows [item_lo, item_hi) are contiguous in the table, class after class: the two-ahead
                    // prefetch of the row entries runs straight through the class boundaries (the table is padded
                    // at its end, so it may also run past item_hi)
                    const uint16_t* __restrict__ ent =
                        x.cls_entries + (static_cast<size_t>(tile.group_base) + static_cast<size_t>(item_lo)) * 32 + lane;
                    int pos = ent[0], pos1 = ent[32];
                    for (int q = 0; q < 16; ++q) {
                        const int ra = max(item_lo, s_off[q]), rb = min(item_hi, s_off[q + 1]);
                        if (ra >= rb) continue;  // this warp owns no row of class q
                        float2 acc2[G];  // {bucket 0, bucket 1} per column pair: one FADD2 per gathered slot
#pragma unroll
                        for (int g = 0; g < G; ++g) acc2[g] = make_float2(0.f, 0.f);
                        for (int it = ra; it < rb; ++it) {
                            ent += 32;
                            const int pos2 = ent[32];
                            const float2* zp = zbuf + pos;
#pragma unroll
                            for (int g = 0; g < G; ++g) acc2[g] = f2_add(acc2[g], zp[-2 * g]);
                            pos = pos1;
                            pos1 = pos2;
                        }
                        float acc[NV];
#pragma unroll
                        for (int g = 0; g < NV; ++g) acc[g] = 0.f;
#pragma unroll
                        for (int g = 0; g < G; ++g) {
                            acc[g] = acc2[g].x;
                            acc[G + g] = acc2[g].y;
                        }
                        const float sum = warp_transpose_sum<NV>(acc, lane);
                        // lane L holds value (L*NV)>>5: value index v -> bucket v / G, pair v % G
                        if (NV == 32 || (lane & 1) == 0) cpart[(warp + q) * NV + ((lane * NV) >> 5)] = sum;
                    }
                }
                __syncthreads();
                PM_PHASE(3);  // M-step gather (+ wait)
                // class sums of the tile, per-warp partials added in warp order (deterministic)
                {
                    #pragma unroll 1
                    for (int e = threadIdx.x; e < 32 * G; e += blockDim.x) {
                        const int b = e / (16 * G), rem = e - b * 16 * G;
                        const int q = rem / G, g = rem - q * G;
                        // the warps owning rows of class q are consecutive: start at the one holding the class's first
                        // row (closed-form guess, corrected against wrow) and walk while rows remain
                        const int q_lo = s_off[q], q_hi = s_off[q + 1];
                        int w = min(static_cast<int>(static_cast<long long>(q_lo) * nwarps / max(s_off[16], 1)), nwarps - 1);
                        while (w > 0 && wrow[w] > q_lo) --w;
                        while (w + 1 < nwarps && wrow[w + 1] <= q_lo) ++w;
                        float sum = 0.f;
                        #pragma unroll 1
                        for (; w < nwarps && wrow[w] < q_hi; ++w) {
                            if (max(wrow[w], q_lo) < min(wrow[w + 1], q_hi)) sum += cpart[(w + q) * NV + b * G + g];
                        }
                        Cq[e] += sum;
                    }
                }
                if (tile_i + 1 < x.n_tiles) __syncthreads();  // z buffer, s_off and cpart are reused by the next tile
            }  // tiles
            if (final_pass) break;
            if (lane == 0) {
                llpart[warp * 2 + 0] = ll0;
                llpart[warp * 2 + 1] = ll1;
            }
            __syncthreads();
            // marginalise to motif counts, then write_column (refine.hpp:241-269) in FP64.
            // Thread e = 4c + r owns theta cell (column c, symbol r); c == l is the background column.
            // The four lanes of a column exchange their values with shuffles.  A frozen bucket keeps its theta.
            ++iterations;
            const int nw_m = (4 * l + 31) >> 5;  // warps covering the 4l motif cells of one bucket
            if (nwarps >= 2 * nw_m + 2) {
                // both buckets at once: warps [bb*nw_m, (bb+1)*nw_m) own bucket bb's motif cells, warp 2*nw_m + bb
                // its background column (all 32 lanes share the l column sums, then lanes 0..3 normalise)
                const bool bg_warp = warp >= 2 * nw_m && warp < 2 * nw_m + 2;
                const int bb = bg_warp ? warp - 2 * nw_m : (warp < nw_m ? 0 : 1);
                if (warp < 2 * nw_m + 2 && !(bb ? stop1 : stop0)) {
                    const float* C = Cq + bb * 16 * G;
                    const int e = bg_warp ? lane : static_cast<int>(threadIdx.x) - bb * nw_m * 32;
                    const int r = e & 3;
                    bool live;
                    int cell;
                    double raw;
                    if (!bg_warp) {
                        live = e < 4 * l;
                        const int c = live ? e >> 2 : 0, g = c >> 1;
                        cell = (c + 1) * 4 + r;
                        raw = 0.0;
                        for (int o = 0; o < 4; ++o) raw += static_cast<double>(C[((c & 1) ? (4 * o + r) : (4 * r + o)) * G + g]);
                    } else {
                        // background = symbol totals - expected motif counts, clamped at 0
                        live = lane < 4;
                        cell = r;
                        double cnt = 0.0;
                        #pragma unroll 1
                        for (int cc = lane >> 2; cc < l; cc += 8) {
                            const int g = cc >> 1;
                            for (int o = 0; o < 4; ++o) cnt += static_cast<double>(C[((cc & 1) ? (4 * o + r) : (4 * r + o)) * G + g]);
                        }
                        cnt += __shfl_xor_sync(0xffffffffu, cnt, 4);
                        cnt += __shfl_xor_sync(0xffffffffu, cnt, 8);
                        cnt += __shfl_xor_sync(0xffffffffu, cnt, 16);
                        raw = fmax(p.tot_sym[r] - cnt, 0.0);
                    }
                    double sum = raw + __shfl_xor_sync(0xffffffffu, raw, 1);
                    sum += __shfl_xor_sync(0xffffffffu, sum, 2);
                    const double v = sum > 0.0 ? fmax(raw / sum, 1e-9) : 0.25;
                    double fs = v + __shfl_xor_sync(0xffffffffu, v, 1);
                    fs += __shfl_xor_sync(0xffffffffu, fs, 2);
                    if (live) {
                        const double tv = v / fs;
                        thd[bb * TH + cell] = tv;
                        L64[bb * TH + cell] = log_f64(fmax(tv, 1e-9));
                    }
                }
            } else {
            for (int bb = 0; bb < 2; ++bb) {
                if (bb ? stop1 : stop0) continue;
                if (warp < (TH + 31) / 32) {
                    const float* C = Cq + bb * 16 * G;
                    const int e = threadIdx.x;
                    const bool live = e < TH;
                    const int c = live ? e >> 2 : 0, r = e & 3;
                    double raw;
                    if (c < l) {
                        const int g = c >> 1;
                        raw = 0.0;
                        for (int o = 0; o < 4; ++o) raw += static_cast<double>(C[((c & 1) ? (4 * o + r) : (4 * r + o)) * G + g]);
                    } else {
                        // background = symbol totals - expected motif counts, clamped at 0
                        double bg = p.tot_sym[r];
                        #pragma unroll 1
                        for (int cc = 0; cc < l; ++cc) {
                            const int g = cc >> 1;
                            double cnt = 0.0;
                            for (int o = 0; o < 4; ++o) cnt += static_cast<double>(C[((cc & 1) ? (4 * o + r) : (4 * r + o)) * G + g]);
                            bg -= cnt;
                        }
                        raw = fmax(bg, 0.0);
                    }
                    double sum = raw + __shfl_xor_sync(0xffffffffu, raw, 1);
                    sum += __shfl_xor_sync(0xffffffffu, sum, 2);
                    const double v = sum > 0.0 ? fmax(raw / sum, 1e-9) : 0.25;
                    double fs = v + __shfl_xor_sync(0xffffffffu, v, 1);
                    fs += __shfl_xor_sync(0xffffffffu, fs, 2);
                    if (live) {
                        const double tv = v / fs;
                        thd[bb * TH + (c < l ? c + 1 : 0) * 4 + r] = tv;
                        L64[bb * TH + (c < l ? c + 1 : 0) * 4 + r] = log_f64(fmax(tv, 1e-9));
                    }
                }
            }
            }
            if (threadIdx.x >= blockDim.x - 2) {
                const int bb = threadIdx.x - (blockDim.x - 2);
                if (!(bb ? stop1 : stop0)) {
                    // sum_i (log prod theta_bg - log W_i) + sum_i logsumexp_i
                    double ll = 0.0;
                    for (int r = 0; r < 4; ++r) ll += p.tot_sym[r] * dscal[bb * 6 + 2 + r];
                    ll -= sum_logw;
                    for (int w = 0; w < nwarps; ++w) ll += llpart[w * 2 + bb];
                    if (p.out_ll && (bb == 0 || live1)) p.out_ll[static_cast<int64_t>(ois[bb]) * p.max_iters + (iterations - 1)] = ll;
                    iscal[bb * 4 + 0] = (iterations >= 2 && ll - dscal[bb * 6] < p.tol) ? 1 : 0;  // refine.hpp:296-304
                    // The likelihood is FP64-accurate where EM has saturated and carries FP32 sums elsewhere (<= ~2e-5): a
                    // gain this close to tol is decided by the FP64 kernel instead (the last iteration cannot stop the loop).
                    if (p.flag_exact && iterations >= 2 && iterations < p.max_iters && fabs((ll - dscal[bb * 6]) - p.tol) <= 1e-4 &&
                        (bb == 0 || live1))
                        p.flag_exact[ois[bb]] = 1;
                    iscal[bb * 4 + 3] = iterations;
                    dscal[bb * 6] = ll;
                }
            }
            __syncthreads();
            PM_PHASE(4);  // class-sum reduce, theta update, LL
            stop0 = iscal[0] != 0;
            stop1 = iscal[4] != 0;
            final_pass = iterations >= p.max_iters || (stop0 && stop1);
        }

        // ---- score / consensus over the argmax rows (scoring.hpp:84-126), expectation (refine.hpp:130-136)
        __syncthreads();
        PM_PHASE(5);  // final E-step sweep (positions)
        if (threadIdx.x < 64 && (threadIdx.x & 31) < l) {
            const int bb = threadIdx.x >> 5, c = threadIdx.x & 31;
            const int* pc = prof + bb * 128 + c * 4;
            int best = 0;
            for (int r = 1; r < 4; ++r) {
                if (pc[r] > pc[best]) best = r;
            }
            atomicAdd(&iscal[bb * 4 + 1], pc[best]);
            atomicOr(&cons_bits[bb], static_cast<unsigned long long>(best) << (62 - 2 * c));
        }
        __syncthreads();
        if (threadIdx.x < 2 && (threadIdx.x == 0 || live1)) {
            const int bb = threadIdx.x;
            const unsigned int wi = ois[bb];
            double ex = 0.0;
            #pragma unroll 1
            for (int c = 1; c <= l; ++c) {
                const double* tc = thd + bb * TH + c * 4;
                ex += fmax(fmax(tc[0], tc[1]), fmax(tc[2], tc[3]));
            }
            p.out_score[wi] = iscal[bb * 4 + 1];
            p.out_iters[wi] = iscal[bb * 4 + 3];
            p.out_exp[wi] = ex;
            p.out_cons[wi] = cons_bits[bb];
            atomicAdd(p.iter_total, static_cast<unsigned long long>(iscal[bb * 4 + 3] + 1));
            if (iscal[bb * 4 + 2]) atomicExch(p.error_flag, 1u);
        }
        if (p.out_theta) {
            #pragma unroll 1
            for (int e2 = threadIdx.x; e2 < 2 * TH; e2 += blockDim.x) {
                const int bb = e2 >= TH, e = e2 - bb * TH;
                if (bb && !live1) continue;
                const int c = e >> 2, r = e & 3;
                p.out_theta[static_cast<int64_t>(ois[bb]) * 4 * (l + 1) + r * (l + 1) + c] = thd[e2];
            }
        }
        PM_PHASE(6);  // score, consensus, outputs
    }
    // no bulk copy may still be in flight into this CTA's shared memory when it exits
    if (big) {
        if (x.n_tiles > 1) {
            mbar_wait(&mbar[visit & 1], (visit >> 1) & 1);
        } else if (visit == 0) {
            mbar_wait(&mbar[0], 0);
        }
    }
}

}  // namespace k
}  // namespace pm
