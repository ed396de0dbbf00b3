// pm_em_f64.cuh — refine() of one bucket per CTA entirely in FP64, in the reference's own operation order where the
// order is observable (refine.hpp:90-326): per-window weights are summed column by column, the per-sequence maximum
// is exact, write_column sums its four entries in symbol order.  A warp takes a sequence; sums over its windows are
// fixed-shape trees (per-lane strided partial sums, then shuffles: deterministic, a few ulps from the reference's
// sequential sums); the per-sequence likelihood terms are added in sequence order like the reference.
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

__global__ void __launch_bounds__(kF64Threads) em_refine_f64_kernel(const EmParams p, const F64Extra x) {
    __shared__ double th[4 * 32];     // theta[r][c] at c * 4 + r, c = 0 background
    __shared__ double D[4 * 32];      // log max(theta[r][c+1],1e-9) - log max(theta[r][0],1e-9) at c * 4 + r
    __shared__ double lbg[4];
    __shared__ double cnt[4 * 32];                        // M-step counts, cell c * 4 + r
    __shared__ double part[(kF64Threads / 32) * 32 * 4];  // per-warp partial counts
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
                    double se = 0.0;
                    for (int j = lane; j < W; j += 32) {
                        const double e = exp(zi[j] - M);
                        zi[j] = e;
                        se += e;
                    }
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) se += __shfl_xor_sync(0xffffffffu, se, o);
                    const double S = se;
                    if (!final_pass) {
                        for (int j = lane; j < W; j += 32) zi[j] /= S;
                        // log P(S_i) = log prod theta_bg - log W + logsumexp (refine.hpp:200)
                        double lb = 0.0;
                        for (int r = 0; r < 4; ++r) lb += static_cast<double>(p.seq_sym[i * 4 + r]) * lbg[r];
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

            // ---- M-step (refine.hpp:227-237): counts[c][r] = sum of z over the windows that show r at column c.
            // Warp w takes the sequences i = w, w + 20, ...; lane = motif column, four accumulators (one per symbol);
            // the per-warp partials are added in warp order: fixed shape, deterministic.
            __syncthreads();
            {
                const int warp = tid >> 5, lane = tid & 31;
                double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
                for (int i = warp; i < t; i += kF64Threads / 32) {
                    const uint64_t* __restrict__ wp = p.words + p.word_off[i];
                    const int W = p.seq_len[i] - l + 1;
                    const double* zi = z + p.win_off[i];
                    // lane's column of window j is base j + lane: one symbol stream per lane, read word by word
                    const int q0 = lane;  // first base this lane looks at
                    uint64_t word = wp[q0 >> 5];
                    int in_word = q0 & 31;
                    // eight responsibilities are fetched at a time (the loads were the latency of this loop: one L2 round
                    // trip per window); they are added in window order, like the reference's sequential sums
                    for (int j0 = 0; j0 < W; j0 += 8) {
                        double zb[8];
#pragma unroll
                        for (int u = 0; u < 8; ++u) zb[u] = j0 + u < W ? zi[j0 + u] : 0.0;
#pragma unroll
                        for (int u = 0; u < 8; ++u) {
                            if (j0 + u >= W) break;
                            const double zj = zb[u];
                            const unsigned sym = static_cast<unsigned>(word >> (62 - 2 * in_word)) & 3u;
                            if (++in_word == 32) {
                                in_word = 0;
                                word = wp[((q0 + j0 + u + 1) >> 5)];
                            }
                            a0 += sym == 0u ? zj : 0.0;
                            a1 += sym == 1u ? zj : 0.0;
                            a2 += sym == 2u ? zj : 0.0;
                            a3 += sym == 3u ? zj : 0.0;
                        }
                    }
                }
                if (lane < l) {
                    double* out = part + (warp * 32 + lane) * 4;
                    out[0] = a0, out[1] = a1, out[2] = a2, out[3] = a3;
                }
            }
            __syncthreads();
            if (tid < 4 * l) {
                const int c = tid >> 2, r = tid & 3;
                double sum = 0.0;
                for (int w = 0; w < kF64Threads / 32; ++w) sum += part[(w * 32 + c) * 4 + r];
                cnt[tid] = sum;
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
