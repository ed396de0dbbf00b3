// pm_em_smem.cuh — EM refinement kernel for sequence sets whose per-window responsibilities fit in
// shared memory (sum of sequence lengths <= ~50k bases: every t=20 config of BASELINE.json).
//
// One CTA per enriched bucket (persistent grid-stride over the work list), warps stride over
// sequences for the E-step, then over pair-class position groups for the M-step.
//
//   E-step (lane = window)   w_j = sum_g T[g][nibble g of window j]  (pair-symbol log-odds table in smem),
//                            pass A stores w_j and the per-sequence max, pass B turns them into
//                            e_j = exp(w_j - max) and their sum, pass C scales to z_j = e_j / sum.
//   M-step (lane = position) the pair class q(p) = 4 s_p + s_{p+1} of base position p is a property of the
//                            sequence set, not of the bucket, so the positions of every class are grouped
//                            ONCE per set into warps of 32 with pairwise distinct addresses mod 32.  Column
//                            pair g of window j = p - 2g sees class q(p), hence
//                                C[g][q] = sum_{p in class q} z[p - 2g]
//                            is a conflict-free shared-memory gather into G register accumulators with no
//                            data-dependent accumulator index; counts[a][2g] = sum_b C[g][4a+b] and
//                            counts[b][2g+1] = sum_a C[g][4a+b] follow by marginalising (refine.hpp:227-237).
//   precision                dense scan and counts in FP32; theta, log tables, the M-step normalisation and the
//                            log-likelihood in FP64.  Windows within 2^-30 of the per-sequence maximum weight
//                            are re-evaluated in FP64 (their z, the max and the log-sum-exp), which makes the
//                            1e-6 convergence test of refine.hpp:300 reproducible whenever EM has saturated.
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

template <int G>
__global__ void __launch_bounds__(kEmSmemMaxWarps * 32, 3)
em_refine_smem_kernel(const EmParams p, const EmSmemExtra x) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int nwarps = blockDim.x >> 5;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int l = p.l, t = p.t;

    // ---- shared memory carve-up (doubles first for alignment)
    double* thd = reinterpret_cast<double*>(smem_raw);  // [32][4] theta, column 0 = background
    double* D64 = thd + 128;                            // [32][4] log theta[r][c+1] - log theta[r][0]
    double* llpart = D64 + 128;                         // [nwarps]
    double* dscal = llpart + nwarps;                    // [0] previous LL [2..5] log background
    float* T = reinterpret_cast<float*>(dscal + 6);     // [16][16] pair tables
    float* cpart = T + 256;                             // [nwarps][16][G] per-warp class sums
    float* Cq = cpart + nwarps * 16 * G;                // [16][G]
    int* near_j = reinterpret_cast<int*>(Cq + 16 * G);  // [nwarps][kNearCap]
    int* prof = near_j + nwarps * kNearCap;             // [32][4]
    int* iscal = prof + 128;                            // [0] stop [1] score [2] bad
    int* s_off = iscal + 4;                             // [17] first group of each class (+3 pad)
    unsigned long long* cons_bits = reinterpret_cast<unsigned long long*>(s_off + 20);
    float* mprev_s = reinterpret_cast<float*>(cons_bits + 1);  // [min(t, kMaxFusedSeqs) rounded to even]
    const int n_mprev = t <= kMaxFusedSeqs ? ((t + 1) & ~1) : 0;
    float* zbuf = mprev_s + n_mprev;                    // [max tile zlen]
    float* mprev = n_mprev > 0 ? mprev_s : x.mprev_g + static_cast<size_t>(blockIdx.x) * t;
    // packed words of the current tile (and, with several tiles, of the next one), filled by TMA
    uint64_t* wstage = reinterpret_cast<uint64_t*>(
        (reinterpret_cast<uintptr_t>(zbuf + x.zcap) + 15) & ~static_cast<uintptr_t>(15));
    const int n_stages = x.n_tiles > 1 ? 2 : 1;
    unsigned long long* mbar = reinterpret_cast<unsigned long long*>(wstage + static_cast<size_t>(x.wcap) * n_stages);
    // visit v of the cyclic tile walk uses stage v % n_stages; its data is complete when mbar[stage] has
    // flipped (v / n_stages) & 1 ... tracked as a running visit counter
    unsigned int visit = 0;
    if (threadIdx.x == 0) {
        mbar_init(&mbar[0], 1);
        mbar_init(&mbar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        const TileDesc t0 = x.tiles[0];
        mbar_expect_tx(&mbar[0], static_cast<unsigned>(t0.n_words) * 8u);
        tma_load_1d(wstage, p.words + t0.word_begin, static_cast<unsigned>(t0.n_words) * 8u, &mbar[0]);
    }
    __syncthreads();

    int* my_near = near_j + warp * kNearCap;
    const int colshift = 62 - 2 * lane;

    const unsigned int n_work = p.n_work_dev ? *p.n_work_dev : p.n_work;
    for (unsigned int wi = blockIdx.x; wi < n_work; wi += gridDim.x) {
        const WorkDesc wd = p.work[wi];
        __syncthreads();
#ifdef PM_EM_TIMING
        long long t_phase = clock64();
#endif

        // ---- init_model (refine.hpp:90-127), pseudocount 0
        for (int i = threadIdx.x; i < 128; i += blockDim.x) prof[i] = 0;
        if (threadIdx.x == 0) {
            iscal[0] = 0;
            iscal[2] = 0;
            dscal[0] = 0.0;
        }
        __syncthreads();
        for (unsigned int m = threadIdx.x; m < wd.count; m += blockDim.x) {
            const int64_t f = p.members[wd.mem_begin + m];
            const int i = seq_of_flat(p.win_off, t, f);
            const uint64_t v = load_window(p.words + p.word_off[i], f - p.win_off[i]);
            for (int c = 0; c < l; ++c) atomicAdd(&prof[c * 4 + (static_cast<unsigned>(v >> (62 - 2 * c)) & 3u)], 1);
        }
        __syncthreads();
        for (int e = threadIdx.x; e < 4 * (l + 1); e += blockDim.x) {
            const int c = e >> 2, r = e & 3;
            thd[e] = c == 0 ? p.tot_sym[r] / p.tot_bases
                            : static_cast<double>(prof[(c - 1) * 4 + r]) / static_cast<double>(wd.count);
        }
        __syncthreads();

        int iterations = 0;
        bool final_pass = false;
        PM_PHASE(0);  // init_model
        for (;;) {
            // ---- log tables of the current theta (refine.hpp:155-161), FP64 then rounded once to FP32
            for (int e = threadIdx.x; e < 4 * l; e += blockDim.x) {
                const int c = e >> 2, r = e & 3;
                D64[e] = log(fmax(thd[(c + 1) * 4 + r], 1e-9)) - log(fmax(thd[r], 1e-9));
            }
            if (threadIdx.x >= blockDim.x - 4) {
                const int r = threadIdx.x - (blockDim.x - 4);
                dscal[2 + r] = log(fmax(thd[r], 1e-9));
            }
            if (final_pass) {
                for (int i = threadIdx.x; i < 128; i += blockDim.x) prof[i] = 0;
                if (threadIdx.x == 0) {
                    iscal[1] = 0;
                    *cons_bits = 0ULL;
                }
            }
            __syncthreads();
            for (int e = threadIdx.x; e < 16 * G; e += blockDim.x) {
                const int g = e >> 4, q = e & 15;
                const int c0 = 2 * g, c1 = 2 * g + 1;
                double v = 0.0;
                if (c0 < l) v = D64[c0 * 4 + (q >> 2)];
                if (c1 < l) v += D64[c1 * 4 + (q & 3)];
                T[e] = static_cast<float>(v);
            }
            __syncthreads();

            PM_PHASE(1);  // log tables
            double ll_warp = 0.0;
            for (int e = lane; e < 16 * G; e += 32) cpart[warp * 16 * G + e] = 0.f;  // this warp's class sums
            for (int tile_i = 0; tile_i < x.n_tiles; ++tile_i) {
            const TileDesc tile = x.tiles[tile_i];
            // ---- packed words of this tile: staged by TMA (single tile: once for the whole kernel)
            const uint64_t* __restrict__ wtile = wstage + static_cast<size_t>(x.wcap) * (visit % n_stages);
            if (x.n_tiles > 1) {
                if (threadIdx.x == 0) {  // prefetch the next tile of the cyclic walk into the other stage
                    const TileDesc nt = x.tiles[tile_i + 1 < x.n_tiles ? tile_i + 1 : 0];
                    unsigned long long* nb = &mbar[(visit + 1) & 1];
                    mbar_expect_tx(nb, static_cast<unsigned>(nt.n_words) * 8u);
                    tma_load_1d(wstage + static_cast<size_t>(x.wcap) * ((visit + 1) & 1), p.words + nt.word_begin,
                                static_cast<unsigned>(nt.n_words) * 8u, nb);
                }
                mbar_wait(&mbar[visit & 1], (visit >> 1) & 1);
            } else if (visit == 0) {
                mbar_wait(&mbar[0], 0);
            }
            ++visit;
            // ================= E-step: warp per sequence of the tile =================
            if (threadIdx.x < 17) s_off[threadIdx.x] = x.tile_group_off[tile_i * 17 + threadIdx.x];
            for (int k = threadIdx.x, k_end = x.seq_zoff[tile.seq_begin]; k < k_end; k += blockDim.x) zbuf[k] = 0.f;  // front pad
            for (int i = tile.seq_begin + warp; i < tile.seq_end; i += nwarps) {
                const uint64_t* __restrict__ wp = wtile + (p.word_off[i] - tile.word_begin);
                const int W = p.seq_len[i] - l + 1;
                const int chunks = (W + 31) >> 5;
                float* zs = zbuf + x.seq_zoff[i];
                {
                    // slots that are not window starts (the last l-1 bases and the balancing gap up to the
                    // next sequence) read as zero in the M-step gather
                    const int z_end = (i + 1 < tile.seq_end ? x.seq_zoff[i + 1] : tile.zlen) - x.seq_zoff[i];
                    for (int k = W + lane; k < z_end; k += 32) zs[k] = 0.f;
                }

                // pass A.  From the second iteration on the exp is fused in, taken relative to the
                // previous iteration's maximum of this sequence (softmax is shift-invariant), and the
                // windows within exp(log_eps - kNearMargin) of that maximum are listed on the way.
                constexpr float kNearMargin = 4.f;
                const bool fused = !final_pass && iterations > 0;
                float ref = fused ? mprev[i] : 0.f;
                float best_w = -INFINITY, s_all = 0.f, s_far = 0.f;
                int best_j = 0, nnear = 0;
                bool overflow = false;
                if (fused) {
                    estep_pass_a<G, true, false>(T, wp, W, lane, zs, ref, fast_ex2((p.log_z_eps - kNearMargin) * kLog2e),
                                                 best_w, best_j, s_all, s_far, my_near, nnear, overflow);
                } else if (final_pass) {
                    estep_pass_a<G, false, true>(T, wp, W, lane, zs, 0.f, 0.f, best_w, best_j, s_all, s_far, my_near, nnear, overflow);
                } else {
                    estep_pass_a<G, false, false>(T, wp, W, lane, zs, 0.f, 0.f, best_w, best_j, s_all, s_far, my_near, nnear, overflow);
                }
                const float M = warp_max_f(best_w);
                if (!(M > -INFINITY) || !(M < INFINITY)) iscal[2] = 1;
                __syncwarp();

                if (final_pass) {
                    // ---- positions: per-sequence argmax, ties to the smallest offset (refine.hpp:311-316).
                    // Windows within delta of the FP32 maximum are compared by their FP64 weights.
                    const float delta = 1e-3f + 1e-5f * fabsf(M);
                    for (int c = 0; c < chunks; ++c) {
                        const int j = (c << 5) + lane;
                        const bool keep = j < W && zs[j] >= M - delta;
                        const unsigned ball = __ballot_sync(0xffffffffu, keep);
                        if (ball && !overflow) {
                            if (nnear + __popc(ball) > kNearCap) {
                                overflow = true;
                            } else {
                                if (keep) my_near[nnear + __popc(ball & ((1u << lane) - 1u))] = j;
                                nnear += __popc(ball);
                            }
                        }
                    }
                    __syncwarp();
                    int arg;
                    if (!overflow) {
                        double bw = -INFINITY;
                        int bj = 0x7fffffff;
                        for (int e = lane; e < nnear; e += 32) {
                            const int j = my_near[e];
                            const double w = window_weight_d(D64, load_window(wp, j), l);
                            if (w > bw || (w == bw && j < bj)) {
                                bw = w;
                                bj = j;
                            }
                        }
#pragma unroll
                        for (int o = 16; o > 0; o >>= 1) {
                            const double ow = __shfl_xor_sync(0xffffffffu, bw, o);
                            const int oj = __shfl_xor_sync(0xffffffffu, bj, o);
                            if (ow > bw || (ow == bw && oj < bj)) {
                                bw = ow;
                                bj = oj;
                            }
                        }
                        arg = bj;
                    } else {
#pragma unroll
                        for (int o = 16; o > 0; o >>= 1) {
                            const float ow = __shfl_xor_sync(0xffffffffu, best_w, o);
                            const int oj = __shfl_xor_sync(0xffffffffu, best_j, o);
                            if (ow > best_w || (ow == best_w && oj < best_j)) {
                                best_w = ow;
                                best_j = oj;
                            }
                        }
                        arg = best_j;
                    }
                    if (p.out_pos && lane == 0) p.out_pos[static_cast<int64_t>(wi) * t + i] = arg + 1;
                    if (lane < l) {
                        const uint64_t v = load_window(wp, arg);
                        atomicAdd(&prof[lane * 4 + (static_cast<unsigned>(v >> colshift) & 3u)], 1);
                    }
                    __syncwarp();
                    continue;
                }

                float total = 0.f;
                bool have_e = false;
                if (fused) {
                    total = warp_sum_f(s_all);
                    const float shift = M - ref;
                    have_e = shift > -60.f && shift < 60.f && total > 0.f && total < INFINITY;
                    if (!have_e) {  // the maximum moved too far for FP32 range: redo as two passes
                        best_w = -INFINITY;
                        estep_pass_a<G, false, false>(T, wp, W, lane, zs, 0.f, 0.f, best_w, best_j, s_all, s_far, my_near, nnear, overflow);
                        __syncwarp();
                    }
                }
                // e_j >= near_e  <=>  w_j >= M + log(eps): the windows re-evaluated in FP64
                float near_e;
                if (!have_e) {
                    // first iteration / fallback: e_j = exp(w_j - M), exact near list
                    ref = M;
                    near_e = fast_ex2(p.log_z_eps * kLog2e);
                    s_all = 0.f, s_far = 0.f, nnear = 0, overflow = false;
                    estep_pass_detect<true>(zs, W, lane, M, near_e, s_all, s_far, my_near, nnear, overflow);
                    total = warp_sum_f(s_all);
                } else {
                    near_e = fast_ex2((M - ref + p.log_z_eps) * kLog2e);
                    if (!overflow && M < ref - kNearMargin) {
                        // the maximum dropped by more than the margin: the list may be incomplete, rebuild it
                        float ignore = 0.f;
                        s_far = 0.f, nnear = 0;
                        estep_pass_detect<false>(zs, W, lane, M, near_e, ignore, s_far, my_near, nnear, overflow);
                    }
                }
                if (!(total > 0.f)) iscal[2] = 1;
                const float inv_total = 1.f / total;
                if (lane == 0) mprev[i] = M;
                __syncwarp();
                // listed windows below the exact threshold belong to the far tail after all
                bool near_a = false, near_b = false;
                if (!overflow) {
                    if (lane < nnear) {
                        const float e = zs[my_near[lane]];
                        near_a = e >= near_e;
                        s_far += near_a ? 0.f : e;
                    }
                    if (lane + 32 < nnear) {
                        const float e = zs[my_near[lane + 32]];
                        near_b = e >= near_e;
                        s_far += near_b ? 0.f : e;
                    }
                }
                s_far *= fast_ex2((ref - M) * kLog2e);  // far-tail sum relative to M
                __syncwarp();
                // pass C: z_j = e_j / sum
                for (int c = 0; c < chunks; ++c) {
                    const int j = (c << 5) + lane;
                    if (j < W) zs[j] *= inv_total;
                }
                __syncwarp();

                const unsigned int* sc = p.seq_sym + i * 4;
                const double log_base = sc[0] * dscal[2] + sc[1] * dscal[3] + sc[2] * dscal[4] + sc[3] * dscal[5];
                double lse;  // log sum_j exp(w_j)
                // The FP64 pass is skipped in the last iteration of the budget: its likelihood can no
                // longer stop the loop (refine.hpp:296-304 breaks after max_iters regardless).
                if (!overflow && iterations + 1 < p.max_iters) {
                    // FP64 re-evaluation of the dominant windows; the far tail (each < eps of the
                    // maximum) keeps its FP32 sum
                    const double far = static_cast<double>(warp_sum_f(s_far));
                    double m64 = -INFINITY;
                    double wa = -INFINITY, wb = -INFINITY;
                    if (near_a) wa = window_weight_d(D64, load_window(wp, my_near[lane]), l);
                    if (near_b) wb = window_weight_d(D64, load_window(wp, my_near[lane + 32]), l);
                    m64 = warp_max_d(fmax(wa, wb));
                    wa = near_a ? exp(wa - m64) : 0.0;
                    wb = near_b ? exp(wb - m64) : 0.0;
                    // far * exp(M - m64): |M - m64| ~ 1e-5 and far < W*eps, so first order is exact to ~1e-17
                    const double s64 = warp_sum_d(wa + wb) + far * (1.0 + (static_cast<double>(M) - m64));
                    lse = m64 + log(s64);
                    if (near_a) zs[my_near[lane]] = static_cast<float>(wa / s64);
                    if (near_b) zs[my_near[lane + 32]] = static_cast<float>(wb / s64);
                } else {
                    lse = static_cast<double>(ref) + log(static_cast<double>(total));  // total is relative to ref
                }
                // log P(S_i) = log prod theta_bg - log W + logsumexp_j w_ij   (refine.hpp:200)
                ll_warp += log_base - p.seq_logw[i] + lse;
                __syncwarp();
            }
            if (final_pass) {  // the final sweep has no M-step
                if (tile_i + 1 < x.n_tiles) __syncthreads();  // the next tile reuses the z buffer
                continue;
            }
            __syncthreads();
            PM_PHASE(2);  // E-step (warp 0's sequences + wait for the slowest warp)

            // ================= M-step of the tile: conflict-free class gather =================
            {
                const int total_groups = s_off[16];
                const int item_lo = static_cast<int>(static_cast<long long>(total_groups) * warp / nwarps);
                const int item_hi = static_cast<int>(static_cast<long long>(total_groups) * (warp + 1) / nwarps);
                const uint16_t* __restrict__ rows = x.cls_entries + static_cast<size_t>(tile.group_base) * 32;
                for (int q = 0; q < 16; ++q) {
                    const int a = max(item_lo, s_off[q]), b = min(item_hi, s_off[q + 1]);
                    if (a >= b) continue;  // this warp owns no row of class q
                    float acc[G];
#pragma unroll
                    for (int g = 0; g < G; ++g) acc[g] = 0.f;
                    const uint16_t* __restrict__ ent = rows + static_cast<size_t>(a) * 32 + lane;
                    int pos = ent[0];
                    for (int it = a; it < b; ++it) {
                        ent += 32;
                        const int nxt = it + 1 < b ? static_cast<int>(ent[0]) : 0;  // prefetch the next row
                        const float* zp = zbuf + pos;
#pragma unroll
                        for (int g = 0; g < G; ++g) acc[g] += zp[-2 * g];
                        pos = nxt;
                    }
#pragma unroll
                    for (int g = 0; g < G; ++g) {
                        const float sum = warp_sum_f(acc[g]);
                        if (lane == 0) cpart[(warp * 16 + q) * G + g] += sum;
                    }
                }
            }
            if (tile_i + 1 < x.n_tiles) __syncthreads();  // z buffer and s_off are reused by the next tile
            }  // tiles
            if (final_pass) break;
            if (lane == 0) llpart[warp] = ll_warp;
            __syncthreads();
            PM_PHASE(3);  // M-step gather + flush (+ wait)
            // C[q][g] = sum of the per-warp class sums, in warp order
            for (int e = threadIdx.x; e < 16 * G; e += blockDim.x) {
                float sum = 0.f;
                for (int w = 0; w < nwarps; ++w) sum += cpart[w * 16 * G + e];
                Cq[e] = sum;
            }
            __syncthreads();
            // marginalise to motif counts, then write_column (refine.hpp:241-269) in FP64.
            // Thread e = 4c + r owns theta cell (column c, symbol r); c == l is the background column.
            // The four lanes of a column exchange their values with shuffles.
            if (warp < (4 * (l + 1) + 31) / 32) {
                const int e = threadIdx.x;
                const bool live = e < 4 * (l + 1);
                const int c = live ? e >> 2 : 0, r = e & 3;
                double raw;
                if (c < l) {
                    const int g = c >> 1;
                    raw = 0.0;
                    for (int o = 0; o < 4; ++o) raw += static_cast<double>(Cq[((c & 1) ? (4 * o + r) : (4 * r + o)) * G + g]);
                } else {
                    // background = symbol totals - expected motif counts, clamped at 0
                    double b = p.tot_sym[r];
                    for (int cc = 0; cc < l; ++cc) {
                        const int g = cc >> 1;
                        double cnt = 0.0;
                        for (int o = 0; o < 4; ++o) cnt += static_cast<double>(Cq[((cc & 1) ? (4 * o + r) : (4 * r + o)) * G + g]);
                        b -= cnt;
                    }
                    raw = fmax(b, 0.0);
                }
                double sum = raw + __shfl_xor_sync(0xffffffffu, raw, 1);
                sum += __shfl_xor_sync(0xffffffffu, sum, 2);
                const double v = sum > 0.0 ? fmax(raw / sum, 1e-9) : 0.25;
                double fs = v + __shfl_xor_sync(0xffffffffu, v, 1);
                fs += __shfl_xor_sync(0xffffffffu, fs, 2);
                if (live) thd[(c < l ? c + 1 : 0) * 4 + r] = v / fs;
            }
            ++iterations;
            if (threadIdx.x == 0) {
                double ll = 0.0;
                for (int w = 0; w < nwarps; ++w) ll += llpart[w];
                if (p.out_ll) p.out_ll[static_cast<int64_t>(wi) * p.max_iters + (iterations - 1)] = ll;
                iscal[0] = (iterations >= 2 && ll - dscal[0] < p.tol) ? 1 : 0;  // refine.hpp:296-304
                dscal[0] = ll;
            }
            __syncthreads();
            PM_PHASE(4);  // class-sum reduce, theta update, LL
            final_pass = iscal[0] != 0 || iterations >= p.max_iters;
        }
        PM_PHASE(5);  // final E-step sweep (positions)

        // ---- score / consensus over the argmax rows (scoring.hpp:84-126), expectation (refine.hpp:130-136)
        __syncthreads();
        if (threadIdx.x < l) {
            const int* pc = prof + threadIdx.x * 4;
            int best = 0;
            for (int r = 1; r < 4; ++r) {
                if (pc[r] > pc[best]) best = r;
            }
            atomicAdd(&iscal[1], pc[best]);
            atomicOr(cons_bits, static_cast<unsigned long long>(best) << (62 - 2 * threadIdx.x));
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            double ex = 0.0;
            for (int c = 1; c <= l; ++c) {
                const double* tc = thd + c * 4;
                ex += fmax(fmax(tc[0], tc[1]), fmax(tc[2], tc[3]));
            }
            p.out_score[wi] = iscal[1];
            p.out_iters[wi] = iterations;
            p.out_exp[wi] = ex;
            p.out_cons[wi] = *cons_bits;
            atomicAdd(p.iter_total, static_cast<unsigned long long>(iterations + 1));
            if (iscal[2]) atomicExch(p.error_flag, 1u);
        }
        if (p.out_theta) {
            for (int e = threadIdx.x; e < 4 * (l + 1); e += blockDim.x) {
                const int c = e >> 2, r = e & 3;
                p.out_theta[static_cast<int64_t>(wi) * 4 * (l + 1) + r * (l + 1) + c] = thd[e];
            }
        }
        PM_PHASE(6);  // score, consensus, outputs
    }
    // no bulk copy may still be in flight into this CTA's shared memory when it exits
    if (x.n_tiles > 1) {
        mbar_wait(&mbar[visit & 1], (visit >> 1) & 1);
    } else if (visit == 0) {
        mbar_wait(&mbar[0], 0);
    }
}

}  // namespace k
}  // namespace pm
