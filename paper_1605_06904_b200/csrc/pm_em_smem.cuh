// pm_em_smem.cuh — building blocks shared by the EM kernels that keep a tile's responsibilities in shared memory
// (pm_em_pair.cuh) or in tensor memory (pm_em_tc.cuh): tile descriptors of the class-gather index, TMA bulk-copy
// and mbarrier wrappers, window assembly, warp reductions.
//
//   tiles   A tile is a run of consecutive sequences whose responsibilities fit the z buffer together; it has
//           its own class-group table.  Small sets (every t=20 config) are a single tile; large sets are swept
//           tile by tile with the class sums accumulated across tiles.
//   M-step  The pair class q(p) = 4 s_p + s_{p+1} of base position p is a property of the sequence set, not of
//           the bucket, so the positions of every class are grouped ONCE per set into rows of 32 with pairwise
//           distinct addresses mod 32: C[g][q] = sum_{p in class q} z[p - 2g] is then a conflict-free gather.
#pragma once
#include "pm_kernels.cuh"

namespace pm {
namespace k {

constexpr int kZPad = 64;    // zero entries in front of the first sequence (dummy lanes read 32..63)
constexpr int kNearCap = 64; // near-maximum windows re-evaluated in FP64, per warp

// A tile is a run of consecutive sequences whose responsibilities fit the z buffer together; it has
// its own class-group table.  Small sets (every t=20 config) are a single tile; large sets are
// swept tile by tile with the class sums accumulated across tiles.
struct TileDesc {
    int seq_begin, seq_end;  // sequences [seq_begin, seq_end)
    int zlen;                // z slots used by the tile (front pad + sequences + balancing gaps)
    int group_base;          // first row of the tile in cls_entries
    int n_words;             // packed words of the tile's sequences (even per sequence => 16-byte multiples)
    int64_t word_begin;      // first packed word of the tile
};

struct EmSmemExtra {
    const TileDesc* tiles;
    int n_tiles;
    const uint16_t* cls_entries;  // [rows][32] z slots relative to the tile (dummies 32+lane point at the zero pad)
    const int* tile_group_off;    // [n_tiles][17] first row of each class, relative to group_base
    const int* seq_zoff;          // [t] first z slot of each sequence within its tile
    float* mprev_g;               // [gridDim.x][t] previous per-sequence maxima when t > kMaxFusedSeqs
    int zcap;                     // largest tile zlen (z buffer size)
    int wcap;                     // largest tile n_words (TMA stage size)
};

__device__ __forceinline__ double warp_max_d(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// log-odds of window v under the FP64 table D64[c][r]
__device__ __forceinline__ double window_weight_d(const double* __restrict__ D64, uint64_t v, int l) {
    double w = 0.0;
    for (int c = 0; c < l; ++c) w += D64[c * 4 + (static_cast<unsigned>(v >> (62 - 2 * c)) & 3u)];
    return w;
}

template <int G>
__device__ __forceinline__ float window_weight_tree(const float* __restrict__ T, uint32_t vh, uint32_t vl) {
    float t[G];
#pragma unroll
    for (int g = 0; g < G; ++g) {
        // byte offset of entry (nibble g) in table g: nibble * 4
        const uint32_t off = g < 7   ? (vh >> (26 - 4 * g)) & 0x3Cu
                             : g == 7 ? (vh << 2) & 0x3Cu
                             : g < 15 ? (vl >> (58 - 4 * g)) & 0x3Cu
                                      : (vl << 2) & 0x3Cu;
        t[g] = *reinterpret_cast<const float*>(reinterpret_cast<const char*>(T) + g * 64 + off);
    }
    // pairwise tree: short dependency chains
#pragma unroll
    for (int s = 1; s < G; s <<= 1) {
#pragma unroll
        for (int g = 0; g + s < G; g += 2 * s) t[g] += t[g + s];
    }
    return t[0];
}

// top-aligned 64-bit window of lane `lane` (shift 2*lane) from words hi, lo as two 32-bit halves
__device__ __forceinline__ void window_halves(uint64_t hi, uint64_t lo, int lane, uint32_t& vh, uint32_t& vl) {
    const uint32_t h1 = static_cast<uint32_t>(hi >> 32), h0 = static_cast<uint32_t>(hi);
    const uint32_t l1 = static_cast<uint32_t>(lo >> 32), l0 = static_cast<uint32_t>(lo);
    const int sh = (2 * lane) & 31;
    const bool upper = lane >= 16;
    const uint32_t a = upper ? h0 : h1, b = upper ? l1 : h0, c = upper ? l0 : l1;
    vh = __funnelshift_l(b, a, sh);
    vl = __funnelshift_l(c, b, sh);
}

// ---- TMA 1-D bulk copy global -> shared with mbarrier completion (sm_90+; SASS: UBLKCP)
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void tma_load_1d(void* dst_smem, const void* src_gmem, unsigned bytes, unsigned long long* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst_smem)),
                 "l"(src_gmem), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "LAB_WAIT:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@p bra DONE;\n"
        "bra LAB_WAIT;\n"
        "DONE:\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ float fast_ex2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
constexpr float kLog2e = 1.4426950408889634f;

// Appends the lanes flagged in `ball` (in lane order) to the warp's near-window list.
__device__ __forceinline__ void near_push(unsigned ball, bool keep, int lane, int j, int* __restrict__ my_near,
                                          int& nnear, bool& overflow) {
    if (ball && !overflow) {
        const int cnt = __popc(ball);
        if (nnear + cnt > kNearCap) {
            overflow = true;
        } else {
            if (keep) my_near[nnear + __popc(ball & ((1u << lane) - 1u))] = j;
            nnear += cnt;
        }
    }
}

// E-step pass A over one sequence: window weights w_j (lane = window).
//   kExp = false: stores w_j.
//   kExp = true : stores e_j = exp(w_j - ref) = 2^(w_j log2e - ref2), accumulates their lane sum (s_all) and
//                 the sum of those below near_thr (s_far), and lists the windows with e_j >= near_thr.
//   kArg tracks the lane's first maximum and its offset (final sweep), otherwise only the maximum.
template <int G, bool kExp, bool kArg, bool kTail>
__device__ __forceinline__ void estep_chunk(const float* __restrict__ T, uint32_t vh, uint32_t vl, int j, bool live,
                                            int lane, float* __restrict__ zs, float ref2, float near_thr,
                                            float& best_w, int& best_j, float& s_all, float& s_far,
                                            int* __restrict__ my_near, int& nnear, bool& overflow) {
    float w = -INFINITY;
    bool keep = false;
    if (!kTail || live) {
        w = window_weight_tree<G>(T, vh, vl);
        if (kExp) {
            const float e = fast_ex2(fmaf(w, kLog2e, -ref2));
            zs[j] = e;
            s_all += e;
            keep = e >= near_thr;
            s_far += keep ? 0.f : e;
        } else {
            zs[j] = w;
        }
    }
    if (kArg) {
        if (w > best_w) {  // strict: the earliest offset is kept
            best_w = w;
            best_j = j;
        }
    } else {
        best_w = fmaxf(best_w, w);
    }
    if (kExp) near_push(__ballot_sync(0xffffffffu, keep), keep, lane, j, my_near, nnear, overflow);
}

template <int G, bool kExp, bool kArg>
__device__ __forceinline__ void estep_pass_a(const float* __restrict__ T, const uint64_t* __restrict__ wp, int W,
                                             int lane, float* __restrict__ zs, float ref, float near_thr,
                                             float& best_w, int& best_j, float& s_all, float& s_far,
                                             int* __restrict__ my_near, int& nnear, bool& overflow) {
    const float ref2 = ref * kLog2e;
    const int full = W >> 5;  // chunks in which every lane has a window
    uint64_t hi = wp[0];
    int c = 0;
    for (; c < full; ++c) {
        const uint64_t lo = wp[c + 1];
        uint32_t vh, vl;
        window_halves(hi, lo, lane, vh, vl);
        hi = lo;
        estep_chunk<G, kExp, kArg, false>(T, vh, vl, (c << 5) + lane, true, lane, zs, ref2, near_thr, best_w, best_j,
                                          s_all, s_far, my_near, nnear, overflow);
    }
    if ((W & 31) != 0) {  // ragged tail (warp-uniform branch)
        const int j = (c << 5) + lane;
        uint32_t vh, vl;
        window_halves(hi, wp[c + 1], lane, vh, vl);
        estep_chunk<G, kExp, kArg, true>(T, vh, vl, j, j < W, lane, zs, ref2, near_thr, best_w, best_j, s_all, s_far,
                                         my_near, nnear, overflow);
    }
}

// Sweep over the stored values of one sequence: kFromW turns stored w_j into e_j = exp(w_j - M) first.
// Sums all e_j (s_all) and those below thr (s_far) and lists the windows with e_j >= thr.
template <bool kFromW>
__device__ __forceinline__ void estep_pass_detect(float* __restrict__ zs, int W, int lane, float M, float thr,
                                                  float& s_all, float& s_far, int* __restrict__ my_near, int& nnear,
                                                  bool& overflow) {
    const int chunks = (W + 31) >> 5;
    for (int c = 0; c < chunks; ++c) {
        const int j = (c << 5) + lane;
        float e = 0.f;
        bool keep = false;
        if (j < W) {
            e = zs[j];
            if (kFromW) {
                e = fast_ex2((e - M) * kLog2e);
                zs[j] = e;
            }
            keep = e >= thr;
        }
        s_all += e;
        s_far += keep ? 0.f : e;
        near_push(__ballot_sync(0xffffffffu, keep), keep, lane, j, my_near, nnear, overflow);
    }
}

#ifdef PM_EM_TIMING
#define PM_PHASE(idx)                                                                    \
    do {                                                                                 \
        if (threadIdx.x == 0) {                                                          \
            const long long now_ = clock64();                                            \
            atomicAdd(p.phase_clk + (idx), static_cast<unsigned long long>(now_ - t_phase)); \
            t_phase = now_;                                                              \
        }                                                                                \
    } while (0)
#else
#define PM_PHASE(idx) do {} while (0)
#endif

constexpr int kEmSmemMaxWarps = 10;
constexpr int kMaxFusedSeqs = 1024;  // sequences whose previous per-sequence maximum is kept in smem

}  // namespace k
}  // namespace pm
