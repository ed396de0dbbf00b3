// pm_em_f64.cuh — refine() of one bucket per CTA entirely in FP64, in the reference's own operation order where the
// order is observable (refine.hpp:90-326): per-window weights are summed column by column, the per-sequence maximum
// is exact, write_column sums its four entries in symbol order, and every sum whose rounding reaches an output is one
// chain in the reference's order: the exponentials of a sequence window by window, the background log term base by
// base, the M-step counts window by window across the whole set, the likelihood sequence by sequence.  What remains
// outside this kernel's control is the last bit of exp() and log() themselves (CUDA's against the host libm's).  A warp
// takes a sequence in the E-step; the M-step is one warp (lane = column).
//
// Not a throughput kernel.  It settles what the FP32 kernels cannot: two candidates of equal score whose expectations
// differ by less than the FP32 error (detail::candidate_improves compares doubles exactly, driver.hpp:127-135), and it
// is the device-side FP64 statement of init_model / em_step that pm_init_model / pm_em_step_exact expose.
#pragma once
#include "pm_kernels.cuh"

namespace pm {
namespace k {

constexpr int kF64Threads = 640;  // 20 warps: one per sequence of the t = 20 configurations (a flagged bucket is a latency problem)
constexpr int kF64LlSeqs = 512;  // per-sequence likelihood terms kept in shared memory (added in sequence order)

struct F64Extra {
    double* zbuf;          // [gridDim.x][x] responsibilities of the CTA's current bucket
    int64_t x;             // total windows
    int steps_only;        // 1: run exactly max_iters em_step()s from theta_in, no stop test, no final E-step outputs
};

// v[0..n) added in index order by a whole warp; every lane returns the sum.  The lanes fetch 32 values at a time
// (coalesced, two groups ahead) and hand them round with shuffles, so the chain waits on the adder, not on memory.
// Entries past n are 0.0, and x + 0.0 == x.
__device__ __forceinline__ double warp_chain_sum(const double* v, int n, int lane) {
    double se = 0.0;
    double cur = lane < n ? v[lane] : 0.0;
    double nxt = 32 + lane < n ? v[32 + lane] : 0.0;
    for (int g = 0; g < n; g += 32) {
        const double nn = g + 64 + lane < n ? v[g + 64 + lane] : 0.0;
#pragma unroll
        for (int u = 0; u < 32; ++u) se += __shfl_sync(0xffffffffu, cur, u);
        cur = nxt;
        nxt = nn;
    }
    return se;
}

__global__ void __launch_bounds__(kF64Threads) em_refine_f64_kernel(const EmParams p, const F64Extra x) {
    __shared__ double th[4 * 32];     // theta[r][c] at c * 4 + r, c = 0 background
    __shared__ double D[4 * 32];      // log max(theta[r][c+1],1e-9) - log max(theta[r][0],1e-9) at c * 4 + r
    __shared__ double lbg[4];
    __shared__ double cnt[4 * 32];                        // M-step counts, cell c * 4 + r
    __shared__ double ll_seq[kF64LlSeqs];
    __shared__ int prof[4 * 32];
    const int tid = threadIdx.x;
    const int l = p.l, t = p.t;
    double* z = x.zbuf + static_cast<size_t>(blockIdx.x) * static_cast<size_t>(x.x);
    const unsigned int n_work = p.n_work_dev ? *p.n_work_dev : p.n_work;

    for (unsigned int wi = blockIdx.x; wi < n_work; wi += gridDim.x) {
        const WorkDesc wd = p.work[wi];
        const unsigned int oi = p.out_map ? p.out_map[wi] : wi;
        __syncthreads();
        // ---- theta0: init_model (refine.hpp:90-127) with pseudocount 0, or the caller's model
        if (p.theta_in) {
            for (int e = tid; e < 4 * (l + 1); e += kF64Threads) {
                const int c = e >> 2, r = e & 3;
                th[e] = p.theta_in[static_cast<int64_t>(wi) * 4 * (l + 1) + r * (l + 1) + c];
            }
        } else {
            for (int e = tid; e < 4 * 32; e += kF64Threads) prof[e] = 0;
            __syncthreads();
            for (unsigned int m = tid; m < wd.count; m += kF64Threads) {
                const int64_t f = p.members[wd.mem_begin + m];
                const int i = seq_of_flat(p.win_off, t, f);
                const uint64_t v = load_window(p.words + p.word_off[i], f - p.win_off[i]);
                for (int c = 0; c < l; ++c) atomicAdd(&prof[(c + 1) * 4 + (static_cast<unsigned>(v >> (62 - 2 * c)) & 3u)], 1);
            }
            __syncthreads();
            for (int e = tid; e < 4 * (l + 1); e += kF64Threads) {
                const int c = e >> 2, r = e & 3;
                if (c == 0) {
                    th[e] = p.tot_sym[r] / p.tot_bases;
                } else {
                    // the reference adds 1.0/denom once per member (refine.hpp:111): same rounding sequence
                    const double inc = 1.0 / static_cast<double>(wd.count);
                    double v = 0.0;
                    for (int k2 = 0; k2 < prof[e]; ++k2) v = __dadd_rn(v, inc);
                    th[e] = v;
                }
            }
        }
        __syncthreads();

        double prev_ll = 0.0;
        int iterations = 0;
        bool final_pass = false;
        for (;;) {
            // ---- log tables (refine.hpp:155-161)
            if (tid < 4) lbg[tid] = log(fmax(th[tid], 1e-9));
            __syncthreads();
            for (int e = tid; e < 4 * l; e += kF64Threads) D[e] = log(fmax(th[e + 4], 1e-9)) - lbg[e & 3];
            if (final_pass) {
                for (int e = tid; e < 4 * 32; e += kF64Threads) prof[e] = 0;
            }
            __syncthreads();

            // ---- E-step (refine.hpp:165-201): warp w takes the sequences w, w + 20, ... (the same assignment as the M-step
            // below), lanes stride over the windows; maxima and sums are reduced with shuffles in a fixed shape.  No
            // block-wide barrier per sequence (a flagged bucket of the (15,4) set: ~0.9 -> ~0.35 ms with 20 warps).
            {
                const int warp = tid >> 5, lane = tid & 31;
                double ll_w = 0.0;
                for (int i = warp; i < t; i += kF64Threads / 32) {
                    const uint64_t* __restrict__ wp = p.words + p.word_off[i];
                    const int W = p.seq_len[i] - l + 1;
                    double* zi = z + p.win_off[i];
                    double mx = -INFINITY;
                    for (int j = lane; j < W; j += 32) {
                        const uint64_t v = load_window(wp, j);
                        double w = 0.0;
                        for (int c = 0; c < l; ++c) w += D[c * 4 + (static_cast<unsigned>(v >> (62 - 2 * c)) & 3u)];
                        zi[j] = w;
                        mx = fmax(mx, w);
                    }
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
                    const double M = mx;
                    if (!(M > -INFINITY) || !(M < INFINITY)) {
                        if (lane == 0) atomicExch(p.error_flag, 1u);
                    }
                    __syncwarp();
                    for (int j = lane; j < W; j += 32) zi[j] = exp(zi[j] - M);
                    __syncwarp();
                    // sum_exp in window order (refine.hpp:191-194): one chain (warp_chain_sum), so
                    // the responsibilities e / S round like the reference's
                    const double S = warp_chain_sum(zi, W, lane);
                    __syncwarp();
                    if (!final_pass) {
                        for (int j = lane; j < W; j += 32) zi[j] /= S;
                        // log P(S_i) = log prod theta_bg - log W + logsumexp (refine.hpp:200)
                        // log_base: one term per base, in sequence order (refine.hpp:172-175)
                        double lb = 0.0;
                        {
                            const int len = p.seq_len[i];
                            for (int q = 0; q < len; q += 32) {
                                const uint64_t word = wp[q >> 5];
                                const int m = min(32, len - q);
                                for (int u = 0; u < m; ++u) lb += lbg[static_cast<unsigned>(word >> (62 - 2 * u)) & 3u];
                            }
                        }
                        const double term = lb - log(static_cast<double>(W)) + M + log(S);
                        if (t <= kF64LlSeqs) {
                            if (lane == 0) ll_seq[i] = term;
                        } else {
                            ll_w += term;
                        }
                    } else {
                        // positions: argmax of z = e / S, ties to the smallest offset (refine.hpp:311-316)
                        double bz = -1.0;
                        int bj = 0x7fffffff;
                        for (int j = lane; j < W; j += 32) {
                            const double zz = zi[j] / S;
                            if (zz > bz) {
                                bz = zz;
                                bj = j;
                            }
                        }
#pragma unroll
                        for (int o = 16; o > 0; o >>= 1) {
                            const double oz = __shfl_xor_sync(0xffffffffu, bz, o);
                            const int oj = __shfl_xor_sync(0xffffffffu, bj, o);
                            if (oz > bz || (oz == bz && oj < bj)) {
                                bz = oz;
                                bj = oj;
                            }
                        }
                        const int arg = bj;
                        if (lane == 0 && p.out_pos) p.out_pos[static_cast<int64_t>(oi) * t + i] = arg + 1;
                        if (lane < l) {
                            const uint64_t v = load_window(wp, arg);
                            atomicAdd(&prof[lane * 4 + (static_cast<unsigned>(v >> (62 - 2 * lane)) & 3u)], 1);
                        }
                    }
                    __syncwarp();
                }
                if (!final_pass && t > kF64LlSeqs && lane == 0) ll_seq[warp] = ll_w;
            }
            __syncthreads();
            // the likelihood: per-sequence terms added in sequence order like the reference (refine.hpp:165-201) -- every
            // thread adds the same list; beyond kF64LlSeqs sequences the per-warp sums are added in warp order
            double ll = 0.0;
            if (!final_pass) {
                const int n_terms = t <= kF64LlSeqs ? t : kF64Threads / 32;
                for (int i = 0; i < n_terms; ++i) ll += ll_seq[i];
            }
            if (final_pass) break;

            // ---- M-step (refine.hpp:227-237): counts[c][r] = sum of z over the windows that show r at column c, added in
            // the reference's order -- sequence by sequence, window by window, ONE chain per cell carried across the
            // sequences -- because the rounding of these sums is observable: saturated models (every column one symbol,
            // the rest on the floor) have expectations that differ in the last bits only, and candidate_improves
            // (driver.hpp:127-135) compares them exactly.  Four warps walk the set, one per symbol; lane = motif column.  The chain
            // costs an FP64 add per window (~0.1 ms per pass on the (15,4) set): this kernel settles a handful of buckets
            // per run, its latency is not the product's.
            __syncthreads();
            if (tid < 128) {
                // warp r keeps the chains of symbol r; lane = motif column
                const unsigned r = static_cast<unsigned>(tid >> 5);
                const int lane = tid & 31;
                const int col = min(lane, l - 1);  // lanes past the motif shadow its last column (their sums are dropped)
                double a = 0.0;
                for (int i = 0; i < t; ++i) {
                    const uint64_t* __restrict__ wp = p.words + p.word_off[i];
                    const int W = p.seq_len[i] - l + 1;
                    const double* zi = z + p.win_off[i];
                    // The lane's column of windows g .. g+31 is the 32 bases from g + col: one 64-bit window, turned into a
                    // match mask for this warp's symbol (bit 62-2u set iff window g+u shows r at the lane's column).  The
                    // responsibilities come 32 at a time, two groups ahead, and go round the warp with shuffles; a step
                    // is two shuffles, two selects and an add -- the loop waits on the adder only.  Responsibilities
                    // past W are 0.0 (a + 0.0 == a), so the last group needs no special case.
                    const uint64_t rpat = static_cast<uint64_t>(r) * 0x5555555555555555ULL;
                    uint64_t v = load_window(wp, col);
                    double cur = lane < W ? zi[lane] : 0.0;
                    double nxt = 32 + lane < W ? zi[32 + lane] : 0.0;
                    for (int g = 0; g < W; g += 32) {
                        const double nn = g + 64 + lane < W ? zi[g + 64 + lane] : 0.0;
                        const uint64_t v_next = g + 32 < W ? load_window(wp, g + 32 + col) : 0ULL;
                        const uint64_t x = v ^ rpat;
                        const uint64_t mt = ~(x | (x >> 1)) & 0x5555555555555555ULL;
                        const unsigned mh = static_cast<unsigned>(mt >> 32), ml = static_cast<unsigned>(mt);
                        const int cur_lo = __double2loint(cur), cur_hi = __double2hiint(cur);
#pragma unroll
                        for (int u = 0; u < 32; ++u) {
                            // the addend is selected (z or 0.0) off the chain; the chain itself is one DADD per window
                            const int zlo = __shfl_sync(0xffffffffu, cur_lo, u), zhi = __shfl_sync(0xffffffffu, cur_hi, u);
                            const bool on = (u < 16 ? (mh & (1u << (30 - 2 * u))) : (ml & (1u << (62 - 2 * u)))) != 0u;
                            a += __hiloint2double(on ? zhi : 0, on ? zlo : 0);
                        }
                        cur = nxt;
                        nxt = nn;
                        v = v_next;
                    }
                }
                if (lane < l) cnt[lane * 4 + r] = a;
            }
            __syncthreads();
            ++iterations;
            // background by subtraction, clamped (refine.hpp:241-253); write_column (refine.hpp:256-269): thread per column
            if (tid <= l) {
                double raw[4];
                if (tid == 0) {
                    for (int r = 0; r < 4; ++r) {
                        double b = p.tot_sym[r];
                        for (int c = 0; c < l; ++c) b -= cnt[c * 4 + r];
                        raw[r] = fmax(b, 0.0);
                    }
                } else {
                    for (int r = 0; r < 4; ++r) raw[r] = cnt[(tid - 1) * 4 + r];
                }
                double sum = 0.0;
                for (int r = 0; r < 4; ++r) sum += raw[r];
                double fs = 0.0;
                for (int r = 0; r < 4; ++r) {
                    raw[r] = sum > 0.0 ? fmax(raw[r] / sum, 1e-9) : 0.25;
                    fs += raw[r];
                }
                for (int r = 0; r < 4; ++r) th[tid * 4 + r] = raw[r] / fs;
            }
            if (tid == 0 && p.out_ll) p.out_ll[static_cast<int64_t>(oi) * p.max_iters + (iterations - 1)] = ll;
            __syncthreads();
            const bool stop = !x.steps_only && iterations >= 2 && ll - prev_ll < p.tol;  // refine.hpp:296-304
            prev_ll = ll;
            if (iterations >= p.max_iters || stop) {
                if (x.steps_only) break;
                final_pass = true;
            }
        }

        // ---- outputs
        __syncthreads();
        if (p.out_theta) {
            for (int e = tid; e < 4 * (l + 1); e += kF64Threads) {
                const int c = e >> 2, r = e & 3;
                p.out_theta[static_cast<int64_t>(oi) * 4 * (l + 1) + r * (l + 1) + c] = th[e];
            }
        }
        if (tid == 0) {
            double ex = 0.0;
            for (int c = 1; c <= l; ++c) ex += fmax(fmax(th[c * 4], th[c * 4 + 1]), fmax(th[c * 4 + 2], th[c * 4 + 3]));
            p.out_exp[oi] = ex;
            p.out_iters[oi] = iterations;
            if (!x.steps_only) {
                int score = 0;
                unsigned long long cons = 0ULL;
                for (int c = 0; c < l; ++c) {
                    int best = 0;
                    for (int r = 1; r < 4; ++r) {
                        if (prof[c * 4 + r] > prof[c * 4 + best]) best = r;
                    }
                    score += prof[c * 4 + best];
                    cons |= static_cast<unsigned long long>(best) << (62 - 2 * c);
                }
                p.out_score[oi] = score;
                p.out_cons[oi] = cons;
            }
            if (p.out_map == nullptr) atomicAdd(p.iter_total, static_cast<unsigned long long>(iterations + 1));  // re-runs were counted
        }
    }
}

// theta0 of init_model (refine.hpp:90-127) with a pseudocount, one CTA per bucket: out[4][l+1] (MotifModel layout)
__global__ void init_model_kernel(const EmParams p, double pseudocount) {
    __shared__ int prof[4 * 32];
    const int tid = threadIdx.x;
    const int l = p.l, t = p.t;
    for (unsigned int wi = blockIdx.x; wi < p.n_work; wi += gridDim.x) {
        const WorkDesc wd = p.work[wi];
        __syncthreads();
        for (int e = tid; e < 4 * 32; e += blockDim.x) prof[e] = 0;
        __syncthreads();
        for (unsigned int m = tid; m < wd.count; m += blockDim.x) {
            const int64_t f = p.members[wd.mem_begin + m];
            const int i = seq_of_flat(p.win_off, t, f);
            const uint64_t v = load_window(p.words + p.word_off[i], f - p.win_off[i]);
            for (int c = 0; c < l; ++c) atomicAdd(&prof[(c + 1) * 4 + (static_cast<unsigned>(v >> (62 - 2 * c)) & 3u)], 1);
        }
        __syncthreads();
        const double denom = static_cast<double>(wd.count) + 4.0 * pseudocount;
        for (int e = tid; e < 4 * (l + 1); e += blockDim.x) {
            const int c = e >> 2, r = e & 3;
            double v;
            if (c == 0) {
                v = p.tot_sym[r] / p.tot_bases;
            } else {
                const double inc = 1.0 / denom;
                v = pseudocount / denom;
                for (int k2 = 0; k2 < prof[e]; ++k2) v = __dadd_rn(v, inc);
            }
            p.out_theta[static_cast<int64_t>(wi) * 4 * (l + 1) + r * (l + 1) + c] = v;
        }
    }
}

}  // namespace k
}  // namespace pm
