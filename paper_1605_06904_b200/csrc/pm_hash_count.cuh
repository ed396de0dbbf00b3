// pm_hash_count.cuh — hash_trial + enriched_buckets for LARGE sets as a device-wide counting sort on the dense
// 4^k table (projection.hpp:258-279 is the reference's own dense backend; :359-390 the enrichment).
//
// What run() uses when a trial does not fit one CTA's shared memory (pm_hash_fused.cuh) and 4^k <= 2^20: the
// 10,000-sequence configuration (x = 9.86 M l-mers per trial).  The radix-sort path moves every (key, index) pair
// through HBM three times; here a pair never exists in memory:
//   count_hist_kernel     thread per l-mer: project it (packed words are L2-resident) and RED.ADD its table entry
//   count_partial/scan    two-level scan over the table in key order: every entry >= s becomes a record
//                         (key, first member slot, size) -- the same key-ordered compaction as the sorted path --
//                         and leaves its first slot behind as the bucket's cursor; every other entry becomes NONE
//   count_scatter_kernel  thread per l-mer: project again; members of enriched buckets take a slot from the cursor
//   count_order_kernel    one CTA per enriched bucket puts its members into ascending l-mer order (the slots were
//                         handed out in arrival order): bitonic sort in shared memory
// Only the members of enriched buckets are ever written (k = 10, s = 19: ~1 % of the l-mers).  Buckets larger than
// kCountMaxBucket (degenerate low-complexity input) make the caller fall back to the radix-sort path.
#pragma once
#include "pm_kernels.cuh"

namespace pm {
namespace k {

constexpr unsigned int kCountNone = 0xFFFFFFFFu;
constexpr int kCountMaxBucket = 4096;   // members one CTA sorts in shared memory
constexpr int kCountScanThreads = 1024;
constexpr int kCountOrderThreads = 128;

struct CountParams {
    const uint64_t* words;
    const int64_t* word_off;
    const int64_t* win_off;
    int t;
    int64_t x, uniform_w;
    int plan_base, n_trials;   // trials of this launch: plans c_plans[0 .. n_trials), tables / outputs at plan_base + tr
    int64_t table_size;        // 4^k
    unsigned int* table;       // [trials][table_size]
};

__device__ __forceinline__ uint64_t count_key_of(const CountParams& p, const PlanProg& pp, int64_t f) {
    int i;
    int64_t j;
    if (p.uniform_w > 0) {  // x fits 32 bits (the reference requires it, projection.hpp:284-287): 32-bit division
        const unsigned int fu = static_cast<unsigned int>(f), w = static_cast<unsigned int>(p.uniform_w);
        i = static_cast<int>(fu / w);
        j = static_cast<int64_t>(fu - static_cast<unsigned int>(i) * w);
    } else {
        i = seq_of_flat(p.win_off, p.t, f);
        j = f - p.win_off[i];
    }
    const uint64_t v = load_window(p.words + p.word_off[i], j);
    uint64_t key = 0;
    const int nruns = pp.nruns;
    for (int r = 0; r < nruns; ++r) {
        const int nb = pp.nbits[r];
        key = (key << nb) | ((v >> pp.rshift[r]) & ((1ULL << nb) - 1ULL));
    }
    return key;
}

__global__ void __launch_bounds__(256) count_hist_kernel(const CountParams p) {
    for (int tr = blockIdx.y; tr < p.n_trials; tr += gridDim.y) {
        const PlanProg& pp = c_plans[tr];
        unsigned int* tab = p.table + static_cast<int64_t>(p.plan_base + tr) * p.table_size;
        for (int64_t f = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; f < p.x;
             f += static_cast<int64_t>(gridDim.x) * blockDim.x) {
            atomicAdd(&tab[count_key_of(p, pp, f)], 1u);  // result unused: a fire-and-forget RED
        }
    }
}

// Exclusive block scan of a pair (records, members) over kCountScanThreads threads.
__device__ __forceinline__ void count_block_scan(unsigned int& a, unsigned int& b, unsigned int* wsum /* [2][32] */,
                                                 unsigned int& tot_a, unsigned int& tot_b) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned int ia = a, ib = b;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned int ua = __shfl_up_sync(0xffffffffu, ia, o), ub = __shfl_up_sync(0xffffffffu, ib, o);
        if (lane >= o) {
            ia += ua;
            ib += ub;
        }
    }
    if (lane == 31) {
        wsum[warp] = ia;
        wsum[32 + warp] = ib;
    }
    __syncthreads();
    if (warp == 0) {
        unsigned int va = wsum[lane], vb = wsum[32 + lane];
        const unsigned int ta = va, tb = vb;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned int ua = __shfl_up_sync(0xffffffffu, va, o), ub = __shfl_up_sync(0xffffffffu, vb, o);
            if (lane >= o) {
                va += ua;
                vb += ub;
            }
        }
        wsum[lane] = va - ta;  // exclusive over warps
        wsum[32 + lane] = vb - tb;
        if (lane == 31) {
            wsum[64] = va;
            wsum[65] = vb;
        }
    }
    __syncthreads();
    const unsigned int ea = ia - a + wsum[warp], eb = ib - b + wsum[32 + warp];
    tot_a = wsum[64];
    tot_b = wsum[65];
    __syncthreads();
    a = ea;
    b = eb;
}

// The scan over the table in key order, two levels: the table of a trial is cut into chunks of kCountChunk keys;
// count_partial_kernel sums (records, members) per chunk, count_scan_kernel gives every chunk the totals of the
// chunks before it (at most 256 pairs to add up) and scans its own keys.  Records come out in ascending key order
// (what the sorted path produces; run() does not depend on the order, the stage API re-sorts by size).
// max_size[0] receives the largest enriched bucket of the launch.
constexpr int kCountItems = 4;
constexpr int kCountChunk = kCountScanThreads * kCountItems;  // 4096 keys per CTA

__global__ void __launch_bounds__(kCountScanThreads) count_partial_kernel(const unsigned int* __restrict__ table, int64_t table_size,
                                                                          int thr, int n_chunks, uint2* __restrict__ partial) {
    __shared__ unsigned int wsum[66];
    const int tr = blockIdx.y, ch = blockIdx.x;
    const unsigned int* tab = table + static_cast<int64_t>(tr) * table_size;
    const int64_t k0 = static_cast<int64_t>(ch) * kCountChunk + static_cast<int64_t>(threadIdx.x) * kCountItems;
    unsigned int nr = 0, nm = 0;
#pragma unroll
    for (int q = 0; q < kCountItems; ++q) {
        const unsigned int cnt = k0 + q < table_size ? tab[k0 + q] : 0u;
        if (cnt >= static_cast<unsigned int>(thr)) {
            ++nr;
            nm += cnt;
        }
    }
    unsigned int tot_r, tot_m;
    count_block_scan(nr, nm, wsum, tot_r, tot_m);
    if (threadIdx.x == 0) partial[static_cast<int64_t>(tr) * n_chunks + ch] = make_uint2(tot_r, tot_m);
}

__global__ void __launch_bounds__(kCountScanThreads) count_scan_kernel(unsigned int* __restrict__ table, int64_t table_size, int thr,
                                                                       int64_t cap_e, int n_chunks, const uint2* __restrict__ partial,
                                                                       uint64_t* __restrict__ rec_key,
                                                                       unsigned int* __restrict__ rec_start,
                                                                       unsigned int* __restrict__ rec_size,
                                                                       unsigned int* __restrict__ n_rec,
                                                                       unsigned int* __restrict__ max_size) {
    __shared__ unsigned int wsum[66];
    __shared__ unsigned int base_sh[2];
    const int tr = blockIdx.y, ch = blockIdx.x;
    unsigned int* tab = table + static_cast<int64_t>(tr) * table_size;
    // totals of the chunks before this one
    {
        unsigned int br = 0, bm = 0;
        for (int c = threadIdx.x; c < ch; c += blockDim.x) {
            const uint2 v = partial[static_cast<int64_t>(tr) * n_chunks + c];
            br += v.x;
            bm += v.y;
        }
        unsigned int tot_r, tot_m;
        count_block_scan(br, bm, wsum, tot_r, tot_m);
        if (threadIdx.x == 0) {
            base_sh[0] = tot_r;
            base_sh[1] = tot_m;
        }
        __syncthreads();
    }
    const int64_t k0 = static_cast<int64_t>(ch) * kCountChunk + static_cast<int64_t>(threadIdx.x) * kCountItems;
    unsigned int cnt[kCountItems];
    unsigned int nr = 0, nm = 0, biggest = 0;
#pragma unroll
    for (int q = 0; q < kCountItems; ++q) {
        cnt[q] = k0 + q < table_size ? tab[k0 + q] : 0u;
        if (cnt[q] >= static_cast<unsigned int>(thr)) {
            ++nr;
            nm += cnt[q];
            biggest = max(biggest, cnt[q]);
        }
    }
    unsigned int tot_r, tot_m;
    count_block_scan(nr, nm, wsum, tot_r, tot_m);
    unsigned int e = base_sh[0] + nr, start = base_sh[1] + nm;
#pragma unroll
    for (int q = 0; q < kCountItems; ++q) {
        if (k0 + q >= table_size) break;
        if (cnt[q] >= static_cast<unsigned int>(thr)) {
            const int64_t o = static_cast<int64_t>(tr) * cap_e + e;
            rec_key[o] = static_cast<uint64_t>(k0 + q);
            rec_start[o] = start;
            rec_size[o] = cnt[q];
            tab[k0 + q] = start;  // the bucket's cursor
            ++e;
            start += cnt[q];
        } else {
            tab[k0 + q] = kCountNone;
        }
    }
    if (ch == n_chunks - 1 && threadIdx.x == 0) n_rec[tr] = base_sh[0] + tot_r;
    biggest = __reduce_max_sync(0xffffffffu, biggest);
    if ((threadIdx.x & 31) == 0 && biggest > 0) atomicMax(max_size, biggest);
}

__global__ void __launch_bounds__(256) count_scatter_kernel(const CountParams p, unsigned int* __restrict__ slots /* [trials][x] */) {
    for (int tr = blockIdx.y; tr < p.n_trials; tr += gridDim.y) {
        const PlanProg& pp = c_plans[tr];
        unsigned int* tab = p.table + static_cast<int64_t>(p.plan_base + tr) * p.table_size;
        unsigned int* out = slots + static_cast<int64_t>(p.plan_base + tr) * p.x;
        for (int64_t f = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; f < p.x;
             f += static_cast<int64_t>(gridDim.x) * blockDim.x) {
            const uint64_t key = count_key_of(p, pp, f);
            // NONE never changes; a cursor only moves within [start, start + size] < x
            if (__ldg(&tab[key]) == kCountNone) continue;
            out[atomicAdd(&tab[key], 1u)] = static_cast<unsigned int>(f);
        }
    }
}

// One CTA per enriched bucket (grid-stride): members into ascending order, in place.
__global__ void __launch_bounds__(kCountOrderThreads) count_order_kernel(unsigned int* __restrict__ slots, int64_t x, int64_t cap_e,
                                                                         int n_trials, const unsigned int* __restrict__ rec_start,
                                                                         const unsigned int* __restrict__ rec_size,
                                                                         const unsigned int* __restrict__ n_rec) {
    __shared__ unsigned int buf[kCountMaxBucket];
    for (int tr = blockIdx.y; tr < n_trials; tr += gridDim.y) {
        const unsigned int ne = n_rec[tr];
        for (unsigned int e = blockIdx.x; e < ne; e += gridDim.x) {
            const int64_t o = static_cast<int64_t>(tr) * cap_e + e;
            const unsigned int n = rec_size[o];
            if (n > static_cast<unsigned int>(kCountMaxBucket)) continue;  // the caller has fallen back already
            unsigned int* seg = slots + static_cast<int64_t>(tr) * x + rec_start[o];
            unsigned int P = 2;
            while (P < n) P <<= 1;
            for (unsigned int i = threadIdx.x; i < P; i += blockDim.x) buf[i] = i < n ? seg[i] : 0xFFFFFFFFu;
            __syncthreads();
            for (unsigned int size = 2; size <= P; size <<= 1) {
                for (unsigned int stride = size >> 1; stride > 0; stride >>= 1) {
                    for (unsigned int i = threadIdx.x; i < (P >> 1); i += blockDim.x) {
                        const unsigned int lo = 2 * i - (i & (stride - 1));  // index with bit `stride` clear
                        const unsigned int hi = lo + stride;
                        const bool up = (lo & size) == 0;
                        const unsigned int a = buf[lo], b = buf[hi];
                        if ((a > b) == up) {
                            buf[lo] = b;
                            buf[hi] = a;
                        }
                    }
                    __syncthreads();
                }
            }
            for (unsigned int i = threadIdx.x; i < n; i += blockDim.x) seg[i] = buf[i];
            __syncthreads();
        }
    }
}

}  // namespace k
}  // namespace pm
