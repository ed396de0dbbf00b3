// pm_kernels.cuh — hand-written sm_100a kernels of the PROJECTION hot path.
//
//   encode_kernel          ASCII -> 2-bit codes packed big-endian into 64-bit words   (alphabet.hpp:33-36)
//   project_keys_kernel    every l-mer of every trial -> projected base-4 key         (projection.hpp:243-254, :332-339)
//   radix_{hist,scan,scatter}  stable segmented LSD radix sort of (key, l-mer index)  (projection.hpp:258-311)
//   enrich_kernel          run detection + stream compaction of buckets of size >= s  (projection.hpp:359-372)
//   work_scan / build_work exclusive scan of per-trial bucket counts -> EM work list
//   em_refine_kernel       one CTA per enriched bucket: init_model, EM, argmax, score (refine.hpp:90-326, scoring.hpp:84-126)
//   (trial_reduce_kernel, the per-trial best candidate, lives in pm_capi.cu next to its record type)
//   hamming_scan_kernel    XOR/popcount distance of a candidate to every window       (sequence.hpp:28-38, oracle.hpp:101-115)
//   score_kernel           profile score / consensus of a start vector                (scoring.hpp:84-126)
//
// Data layout in HBM: sequence i occupies words[word_off[i] .. word_off[i+1]),
// ceil(n_i/32)+1 words (one zero pad word so that word a+1 of any window exists); base p sits at
// bits [62-2(p%32), 64-2(p%32)) of word p/32, i.e. the first base is the most significant digit.
// An l-mer (l <= 31) starting at base j is therefore the top 2l bits of
//   (words[j/32] << 2(j%32)) | (words[j/32+1] >> (64-2(j%32)))
// and a projection keeps runs of adjacent digits in their original significance order.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace pm {
namespace k {

constexpr int kMaxConstPlans = 1024;  // plans resident in constant memory per launch
constexpr int kMaxRuns = 16;          // a plan over l <= 31 positions has at most 16 runs of kept positions

// One projection as an extraction program: run i contributes nbits[i] bits taken at bit
// offset rshift[i] of the top-aligned window word; runs are listed first-kept-first so the
// first kept position ends up as the most significant key digit.
struct PlanProg {
    uint8_t nruns;
    uint8_t keybits;  // 2k
    uint8_t pad[2];
    uint8_t rshift[kMaxRuns];
    uint8_t nbits[kMaxRuns];
};

__constant__ PlanProg c_plans[kMaxConstPlans];

// ---------------------------------------------------------------------------------------------
// small device helpers
// ---------------------------------------------------------------------------------------------
__device__ __forceinline__ uint64_t window_bits(uint64_t hi, uint64_t lo, int sh) {
    // sh = 2*(j%32) in [0,62]
    return sh ? ((hi << sh) | (lo >> (64 - sh))) : hi;
}

// window starting at base j of a sequence whose words start at wp
__device__ __forceinline__ uint64_t load_window(const uint64_t* __restrict__ wp, int64_t j) {
    const int64_t a = j >> 5;
    return window_bits(wp[a], wp[a + 1], 2 * static_cast<int>(j & 31));
}

// index of the sequence owning flat l-mer index f: largest i with win_off[i] <= f
__device__ __forceinline__ int seq_of_flat(const int64_t* __restrict__ win_off, int t, int64_t f) {
    int lo = 0, hi = t;  // invariant: win_off[lo] <= f < win_off[hi]
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (win_off[mid] <= f) lo = mid; else hi = mid;
    }
    return lo;
}

__device__ __forceinline__ int float_order_key(float f) {
    const int i = __float_as_int(f);
    return i ^ ((i >> 31) & 0x7fffffff);
}
__device__ __forceinline__ float float_from_order_key(int i) {
    return __int_as_float(i ^ ((i >> 31) & 0x7fffffff));
}
__device__ __forceinline__ float warp_max_f(float v) {
    return float_from_order_key(__reduce_max_sync(0xffffffffu, float_order_key(v)));
}
__device__ __forceinline__ float warp_sum_f(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// spreads bit i of x to bit 2i
__device__ __forceinline__ uint64_t spread_bits(uint32_t x) {
    uint64_t v = x;
    v = (v | (v << 16)) & 0x0000FFFF0000FFFFULL;
    v = (v | (v << 8)) & 0x00FF00FF00FF00FFULL;
    v = (v | (v << 4)) & 0x0F0F0F0F0F0F0F0FULL;
    v = (v | (v << 2)) & 0x3333333333333333ULL;
    v = (v | (v << 1)) & 0x5555555555555555ULL;
    return v;
}

// ---------------------------------------------------------------------------------------------
// encode: one warp per output word; lane p reads base 32*w+p (coalesced 32 B), the two code bits
// are gathered with ballots and interleaved.  A0 C1 T2 G3 == (ascii >> 1) & 3.
// grid = (ceil(max_words/warps_per_block), t)
// ---------------------------------------------------------------------------------------------
__global__ void encode_kernel(const char* __restrict__ bases, const int64_t* __restrict__ offs,
                              const int64_t* __restrict__ word_off, int t, uint64_t* __restrict__ words,
                              unsigned int* __restrict__ seq_sym /* t x 4 */,
                              unsigned long long* __restrict__ tot_sym /* 4 */,
                              unsigned long long* __restrict__ first_bad /* min flat byte index of a bad symbol */) {
    const int lane = threadIdx.x & 31;
    const int warps_per_block = blockDim.x >> 5;
    for (int i = blockIdx.y; i < t; i += gridDim.y) {
        const int64_t n = offs[i + 1] - offs[i];
        const int64_t nwords = word_off[i + 1] - word_off[i];  // includes the pad word
        for (int64_t w = static_cast<int64_t>(blockIdx.x) * warps_per_block + (threadIdx.x >> 5); w < nwords;
             w += static_cast<int64_t>(gridDim.x) * warps_per_block) {
            const int64_t p = w * 32 + lane;
            const bool in = p < n;
            const unsigned char c = in ? static_cast<unsigned char>(bases[offs[i] + p]) : 'A';
            const bool ok = (c == 'A') | (c == 'C') | (c == 'G') | (c == 'T');
            if (!ok) atomicMin(first_bad, static_cast<unsigned long long>(offs[i] + p));
            const unsigned code = (c >> 1) & 3u;
            const unsigned b0 = __ballot_sync(0xffffffffu, code & 1u);
            const unsigned b1 = __ballot_sync(0xffffffffu, code & 2u);
            const unsigned live = __ballot_sync(0xffffffffu, in);
            if (lane == 0) {
                // lane 0 is the most significant digit: reverse the ballots, then interleave
                words[word_off[i] + w] = (spread_bits(__brev(b1)) << 1) | spread_bits(__brev(b0));
                const unsigned nA = __popc(live & ~b1 & ~b0), nC = __popc(live & ~b1 & b0);
                const unsigned nT = __popc(live & b1 & ~b0), nG = __popc(live & b1 & b0);
                if (live) {
                    atomicAdd(&seq_sym[i * 4 + 0], nA);
                    atomicAdd(&seq_sym[i * 4 + 1], nC);
                    atomicAdd(&seq_sym[i * 4 + 2], nT);
                    atomicAdd(&seq_sym[i * 4 + 3], nG);
                    atomicAdd(&tot_sym[0], static_cast<unsigned long long>(nA));
                    atomicAdd(&tot_sym[1], static_cast<unsigned long long>(nC));
                    atomicAdd(&tot_sym[2], static_cast<unsigned long long>(nT));
                    atomicAdd(&tot_sym[3], static_cast<unsigned long long>(nG));
                }
            }
        }
    }
}

// ---------------------------------------------------------------------------------------------
// projection hashing: thread per l-mer, blockIdx.y = trial within the launch (plan in constant
// memory, so the extraction program is a warp-uniform constant load).
// keys[trial*x + f], idx implicit (first sort pass generates it).
// ---------------------------------------------------------------------------------------------
template <typename KeyT>
__global__ void project_keys_kernel(const uint64_t* __restrict__ words, const int64_t* __restrict__ word_off,
                                    const int64_t* __restrict__ win_off, int t, int64_t x, int64_t uniform_w,
                                    int plan_base, int n_trials, KeyT* __restrict__ keys) {
    for (int tr = blockIdx.y; tr < n_trials; tr += gridDim.y) {
        const PlanProg& pp = c_plans[tr];
        const int nruns = pp.nruns;
        KeyT* out = keys + static_cast<int64_t>(plan_base + tr) * x;
        for (int64_t f = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; f < x;
             f += static_cast<int64_t>(gridDim.x) * blockDim.x) {
            int i;
            int64_t j;
            if (uniform_w > 0) {
                i = static_cast<int>(f / uniform_w);
                j = f - static_cast<int64_t>(i) * uniform_w;
            } else {
                i = seq_of_flat(win_off, t, f);
                j = f - win_off[i];
            }
            const uint64_t v = load_window(words + word_off[i], j);
            uint64_t key = 0;
            for (int r = 0; r < nruns; ++r) {
                const int nb = pp.nbits[r];
                key = (key << nb) | ((v >> pp.rshift[r]) & ((1ULL << nb) - 1ULL));
            }
            out[f] = static_cast<KeyT>(key);
        }
    }
}

// ---------------------------------------------------------------------------------------------
// Stable segmented LSD radix sort, 8-bit digits.  Segment = one trial (stride `seg_stride`
// elements, `seg_len` of them live; seg_len_dev overrides per segment when non-null).
// Tile = 8 warps x 32 lanes x kItems consecutive elements; warp w owns the w-th contiguous
// 32*kItems slice of the tile so that "earlier warp, earlier round, lower lane" is input order.
// ---------------------------------------------------------------------------------------------
constexpr int kSortWarps = 8;
constexpr int kSortItems = 8;
constexpr int kSortTile = kSortWarps * 32 * kSortItems;  // 2048

__device__ __forceinline__ int64_t live_len(int64_t seg_len, const unsigned int* seg_len_dev, int seg) {
    return seg_len_dev ? static_cast<int64_t>(seg_len_dev[seg]) : seg_len;
}

// counts[(seg*256 + digit)*tiles + tile]
template <typename KeyT>
__global__ void __launch_bounds__(kSortWarps * 32)
radix_hist_kernel(const KeyT* __restrict__ keys, int64_t seg_stride, int64_t seg_len,
                  const unsigned int* __restrict__ seg_len_dev, int tiles, int shift,
                  unsigned int* __restrict__ counts) {
    __shared__ unsigned int hist[256];
    const int seg = blockIdx.y, tile = blockIdx.x;
    hist[threadIdx.x] = 0;
    __syncthreads();
    const int64_t n = live_len(seg_len, seg_len_dev, seg);
    const int64_t base = static_cast<int64_t>(tile) * kSortTile;
    const KeyT* in = keys + static_cast<int64_t>(seg) * seg_stride;
#pragma unroll
    for (int it = 0; it < kSortItems; ++it) {
        const int64_t e = base + it * (kSortWarps * 32) + threadIdx.x;
        if (e < n) atomicAdd(&hist[(in[e] >> shift) & 0xFF], 1u);
    }
    __syncthreads();
    counts[(static_cast<int64_t>(seg) * 256 + threadIdx.x) * tiles + tile] = hist[threadIdx.x];
}

// in place: counts -> exclusive offsets within the segment, digit-major then tile.
// grid = segments, block = 256 (thread = digit)
__global__ void __launch_bounds__(256) radix_scan_kernel(unsigned int* __restrict__ counts, int tiles) {
    __shared__ unsigned int totals[256];
    const int seg = blockIdx.x, d = threadIdx.x;
    unsigned int* row = counts + (static_cast<int64_t>(seg) * 256 + d) * tiles;
    unsigned int sum = 0;
    for (int tl = 0; tl < tiles; ++tl) sum += row[tl];
    totals[d] = sum;
    __syncthreads();
    // exclusive scan over 256 digits (Hillis-Steele on shared memory)
    unsigned int v = sum;
    for (int o = 1; o < 256; o <<= 1) {
        const unsigned int add = d >= o ? totals[d - o] : 0u;
        __syncthreads();
        v += add;
        totals[d] = v;
        __syncthreads();
    }
    unsigned int run = v - sum;
    for (int tl = 0; tl < tiles; ++tl) {
        const unsigned int c = row[tl];
        row[tl] = run;
        run += c;
    }
}

// Many-tile variant of the scan (large segments): one CTA per (digit, segment) row scans its tiles in
// place and records the row total; a second kernel turns the 256 totals of a segment into digit
// bases, which the scatter kernel adds (digit_base != nullptr).
__global__ void __launch_bounds__(256) radix_scan_rows_kernel(unsigned int* __restrict__ counts, int tiles,
                                                              unsigned int* __restrict__ totals /* [seg][256] */) {
    __shared__ unsigned int part[256];
    const int d = blockIdx.x, seg = blockIdx.y;
    unsigned int* row = counts + (static_cast<int64_t>(seg) * 256 + d) * tiles;
    const int per = (tiles + 255) / 256;
    const int b = min(tiles, static_cast<int>(threadIdx.x) * per), e = min(tiles, b + per);
    unsigned int sum = 0;
    for (int i = b; i < e; ++i) sum += row[i];
    part[threadIdx.x] = sum;
    __syncthreads();
    unsigned int v = sum;
    for (int o = 1; o < 256; o <<= 1) {
        const unsigned int add = static_cast<int>(threadIdx.x) >= o ? part[threadIdx.x - o] : 0u;
        __syncthreads();
        v += add;
        part[threadIdx.x] = v;
        __syncthreads();
    }
    unsigned int run = v - sum;
    for (int i = b; i < e; ++i) {
        const unsigned int c = row[i];
        row[i] = run;
        run += c;
    }
    if (threadIdx.x == 255) totals[seg * 256 + d] = v;
}

__global__ void __launch_bounds__(256) radix_digit_base_kernel(unsigned int* __restrict__ totals) {
    __shared__ unsigned int part[256];
    unsigned int* row = totals + static_cast<int64_t>(blockIdx.x) * 256;
    const unsigned int mine = row[threadIdx.x];
    part[threadIdx.x] = mine;
    __syncthreads();
    unsigned int v = mine;
    for (int o = 1; o < 256; o <<= 1) {
        const unsigned int add = static_cast<int>(threadIdx.x) >= o ? part[threadIdx.x - o] : 0u;
        __syncthreads();
        v += add;
        part[threadIdx.x] = v;
        __syncthreads();
    }
    row[threadIdx.x] = v - mine;  // exclusive
}

// kFirst: payload of the input is the element's own index within the segment (no idx_in read).
template <typename KeyT, bool kFirst>
__global__ void __launch_bounds__(kSortWarps * 32)
radix_scatter_kernel(const KeyT* __restrict__ keys_in, const unsigned int* __restrict__ idx_in,
                     KeyT* __restrict__ keys_out, unsigned int* __restrict__ idx_out, int64_t seg_stride,
                     int64_t seg_len, const unsigned int* __restrict__ seg_len_dev, int tiles, int shift,
                     const unsigned int* __restrict__ offsets, const unsigned int* __restrict__ digit_base) {
    __shared__ unsigned int warp_cnt[kSortWarps][256];  // per-warp digit counts, then exclusive prefix over warps
    const int seg = blockIdx.y, tile = blockIdx.x;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const unsigned lt_mask = (1u << lane) - 1u;
    for (int i = threadIdx.x; i < kSortWarps * 256; i += blockDim.x) (&warp_cnt[0][0])[i] = 0;
    __syncthreads();

    const int64_t n = live_len(seg_len, seg_len_dev, seg);
    const int64_t seg_base = static_cast<int64_t>(seg) * seg_stride;
    const int64_t wbase = static_cast<int64_t>(tile) * kSortTile + static_cast<int64_t>(warp) * (32 * kSortItems);

    KeyT key[kSortItems];
    unsigned int rank[kSortItems];
#pragma unroll
    for (int it = 0; it < kSortItems; ++it) {
        const int64_t e = wbase + it * 32 + lane;
        const bool live = e < n;
        key[it] = live ? keys_in[seg_base + e] : KeyT(0);
        const unsigned digit = static_cast<unsigned>((key[it] >> shift) & 0xFF);
        // lanes of this warp-round sharing my digit; dead lanes use a private pseudo-digit
        const unsigned peers = __match_any_sync(0xffffffffu, live ? digit : (256u + lane));
        const int leader = __ffs(peers) - 1;
        unsigned int base = 0;
        if (live && lane == leader) {
            base = warp_cnt[warp][digit];
            warp_cnt[warp][digit] = base + __popc(peers);
        }
        base = __shfl_sync(0xffffffffu, base, leader);
        rank[it] = base + __popc(peers & lt_mask);
        __syncwarp();
    }
    __syncthreads();
    // exclusive prefix over warps per digit, plus the tile's global offset for that digit
    for (int d = threadIdx.x; d < 256; d += blockDim.x) {
        unsigned int run = offsets[(static_cast<int64_t>(seg) * 256 + d) * tiles + tile];
        if (digit_base) run += digit_base[seg * 256 + d];
#pragma unroll
        for (int w = 0; w < kSortWarps; ++w) {
            const unsigned int c = warp_cnt[w][d];
            warp_cnt[w][d] = run;
            run += c;
        }
    }
    __syncthreads();
#pragma unroll
    for (int it = 0; it < kSortItems; ++it) {
        const int64_t e = wbase + it * 32 + lane;
        if (e < n) {
            const unsigned digit = static_cast<unsigned>((key[it] >> shift) & 0xFF);
            const int64_t dst = seg_base + warp_cnt[warp][digit] + rank[it];
            keys_out[dst] = key[it];
            idx_out[dst] = kFirst ? static_cast<unsigned int>(e) : idx_in[seg_base + e];
        }
    }
}

// ---------------------------------------------------------------------------------------------
// enrich: CTA (tile, trial) over a tile of the trial's sorted key segment.  An element is the head
// of a bucket when its predecessor has a different key; the bucket is enriched when the key s-1
// places further still matches; its size is an upper-bound search.  Two passes: kWrite = false counts
// the enriched heads of the tile; after an exclusive scan of the tile counts, kWrite = true compacts
// them in key order (block-wide ordered scan: ballot + warp prefix + warp totals) behind the
// tile's offset.  Output per trial (stride cap_e): rec_key, rec_start (segment-relative), rec_size.
// ---------------------------------------------------------------------------------------------
constexpr int kEnrichTile = 8192;

template <typename KeyT, bool kWrite>
__global__ void __launch_bounds__(1024)
enrich_kernel(const KeyT* __restrict__ keys, int64_t x, int s, int64_t cap_e, int etiles,
              unsigned int* __restrict__ tile_cnt /* [trial][etiles]: counts (pass 1) / exclusive offsets (pass 2) */,
              uint64_t* __restrict__ rec_key, unsigned int* __restrict__ rec_start, unsigned int* __restrict__ rec_size) {
    __shared__ unsigned int warp_tot[32];
    __shared__ unsigned int chunk_base;
    const int trial = blockIdx.y, tile = blockIdx.x;
    const KeyT* kk = keys + static_cast<int64_t>(trial) * x;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    if (threadIdx.x == 0) chunk_base = kWrite ? tile_cnt[static_cast<int64_t>(trial) * etiles + tile] : 0u;
    __syncthreads();
    const int64_t t_begin = static_cast<int64_t>(tile) * kEnrichTile;
    const int64_t t_end = min(x, t_begin + kEnrichTile);
    for (int64_t c0 = t_begin; c0 < t_end; c0 += blockDim.x) {
        const int64_t i = c0 + threadIdx.x;
        bool hit = false;
        KeyT key = 0;
        if (i < t_end) {
            key = kk[i];
            const bool head = (i == 0) || (kk[i - 1] != key);
            hit = head && i + s - 1 < x && kk[i + s - 1] == key;
        }
        const unsigned ball = __ballot_sync(0xffffffffu, hit);
        if (lane == 0) warp_tot[warp] = __popc(ball);
        __syncthreads();
        if (kWrite && hit) {
            unsigned int before = chunk_base;
            for (int w = 0; w < warp; ++w) before += warp_tot[w];
            const int64_t e = before + __popc(ball & ((1u << lane) - 1u));
            if (e < cap_e) {
                int64_t lo = i + s - 1, hi = x;  // kk[lo] == key; first index > lo with a different key
                while (hi - lo > 1) {
                    const int64_t mid = (lo + hi) >> 1;
                    if (kk[mid] == key) lo = mid; else hi = mid;
                }
                const int64_t o = static_cast<int64_t>(trial) * cap_e + e;
                rec_key[o] = static_cast<uint64_t>(key);
                rec_start[o] = static_cast<unsigned int>(i);
                rec_size[o] = static_cast<unsigned int>(hi - i);
            }
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            unsigned int tot = chunk_base;
            for (int w = 0; w < nwarps; ++w) tot += warp_tot[w];
            chunk_base = tot;
        }
        __syncthreads();
    }
    if (!kWrite && threadIdx.x == 0) tile_cnt[static_cast<int64_t>(trial) * etiles + tile] = chunk_base;
}

// per trial: tile counts -> exclusive offsets (in place), n_rec[trial] = total.  grid = trials.
__global__ void __launch_bounds__(1024) enrich_scan_kernel(unsigned int* __restrict__ tile_cnt, int etiles,
                                                           unsigned int* __restrict__ n_rec) {
    __shared__ unsigned int part[1024];
    unsigned int* row = tile_cnt + static_cast<int64_t>(blockIdx.x) * etiles;
    const int per = (etiles + blockDim.x - 1) / blockDim.x;
    const int b = min(etiles, static_cast<int>(threadIdx.x) * per), e = min(etiles, b + per);
    unsigned int sum = 0;
    for (int i = b; i < e; ++i) sum += row[i];
    part[threadIdx.x] = sum;
    __syncthreads();
    // Hillis-Steele inclusive scan of the 1024 partials
    unsigned int v = sum;
    for (int o = 1; o < 1024; o <<= 1) {
        const unsigned int add = static_cast<int>(threadIdx.x) >= o ? part[threadIdx.x - o] : 0u;
        __syncthreads();
        v += add;
        part[threadIdx.x] = v;
        __syncthreads();
    }
    unsigned int run = v - sum;
    for (int i = b; i < e; ++i) {
        const unsigned int c = row[i];
        row[i] = run;
        run += c;
    }
    if (threadIdx.x == blockDim.x - 1) n_rec[blockIdx.x] = v;
}

// exclusive scan of n_rec[0..n) -> work_off[0..n], single CTA
__global__ void __launch_bounds__(1024) work_scan_kernel(const unsigned int* __restrict__ n_rec, int n,
                                                         unsigned int* __restrict__ work_off) {
    __shared__ unsigned int part[1024];
    const int per = (n + blockDim.x - 1) / blockDim.x;
    const int b = threadIdx.x * per, e = min(n, b + per);
    unsigned int sum = 0;
    for (int i = b; i < e; ++i) sum += n_rec[i];
    part[threadIdx.x] = sum;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned int run = 0;
        for (int i = 0; i < static_cast<int>(blockDim.x); ++i) {
            const unsigned int c = part[i];
            part[i] = run;
            run += c;
        }
        work_off[n] = run;
    }
    __syncthreads();
    unsigned int run = part[threadIdx.x];
    for (int i = b; i < e; ++i) {
        work_off[i] = run;
        run += n_rec[i];
    }
}

// One EM work item = one enriched bucket.
struct WorkDesc {
    int64_t mem_begin;   // first member in the flat-index array
    uint64_t key;        // projected key (RefinedCandidate.source_bucket)
    unsigned int count;  // members after truncation to r_cap
    int trial;           // trial index within the batch (or bucket index for pm_refine)
};

__global__ void build_work_kernel(const unsigned int* __restrict__ n_rec, const unsigned int* __restrict__ work_off,
                                  const uint64_t* __restrict__ rec_key, const unsigned int* __restrict__ rec_start,
                                  const unsigned int* __restrict__ rec_size, int64_t x, int64_t cap_e, int r_cap,
                                  int n_trials, WorkDesc* __restrict__ work) {
    for (int tr = blockIdx.y; tr < n_trials; tr += gridDim.y) {
        const unsigned int ne = n_rec[tr];
        for (unsigned int e = blockIdx.x * blockDim.x + threadIdx.x; e < ne; e += gridDim.x * blockDim.x) {
            const int64_t o = static_cast<int64_t>(tr) * cap_e + e;
            WorkDesc d;
            d.mem_begin = static_cast<int64_t>(tr) * x + rec_start[o];
            d.key = rec_key[o];
            d.count = min(rec_size[o], static_cast<unsigned int>(r_cap));
            d.trial = tr;
            work[work_off[tr] + e] = d;
        }
    }
}

// ---------------------------------------------------------------------------------------------
// EM refinement: one CTA per bucket (persistent grid-stride over the work list), warps stride
// over sequences.  See DESIGN.md §4.4.
//
//   theta       smem float [l+1][4]   (column 0 = background)
//   pair table  smem float [G][16]    T[g][4a+b] = D[a][2g] + D[b][2g+1],  D[r][c] = log th[r][c+1] - log th[r][0]
//   E-step      lane = window; w = sum_g T[g][nibble g of the window]; warp-uniform running max M,
//               lane-local sum of exp(w-M); windows with w >= M + log(eps) are kept as candidates
//   M-step      lane = column; candidates with z = exp(w-M)/sum >= eps add z to acc[symbol at column]
//               (z below eps are dropped: |d theta| <= W*eps)
// ---------------------------------------------------------------------------------------------
constexpr int kCandCap = 128;  // candidate slots per warp

struct EmParams {
    const uint64_t* words;
    const int64_t* word_off;
    const int32_t* seq_len;
    const int64_t* win_off;
    const unsigned int* seq_sym;  // t x 4
    const double* seq_logw;       // t: log(n_i - l + 1)
    double tot_sym[4];
    double tot_bases;
    int t, l, max_iters;
    double tol;
    float z_eps;
    float log_z_eps;  // -inf when z_eps == 0
    const WorkDesc* work;
    const unsigned int* n_work_dev;  // work count on the device (pm_run) ...
    unsigned int n_work;             // ... or on the host (pm_refine) when n_work_dev == nullptr
    const unsigned int* members;     // flat l-mer indices
    // outputs, indexed by work item
    int32_t* out_score;
    int32_t* out_iters;
    double* out_exp;
    uint64_t* out_cons;    // packed consensus, first base most significant
    int32_t* out_pos;      // [work][t] 1-based or nullptr
    double* out_theta;     // [work][4][l+1] (MotifModel layout) or nullptr
    double* out_ll;        // [work][max_iters] or nullptr
    unsigned long long* iter_total;  // sum over buckets of E-steps executed (iterations + 1)
    unsigned int* error_flag;        // set to 1 on a non-finite window weight (NumericalUnderflowError)
    unsigned long long* phase_clk;   // [8] per-phase clock sums (only with -DPM_EM_TIMING)
    const unsigned int* out_map;     // nullptr, or output slot of each work item (re-runs of flagged buckets, pm_em_tc.cuh)
    const double* theta_in;          // nullptr, or [work][4][l+1] starting models instead of init_model (pm_em_step)
    unsigned char* flag_exact;       // nullptr, or [output slot]: set when a stop decision (refine.hpp:300) fell within the
                                     // error of this kernel's likelihood; the FP64 kernel then refines the bucket again
};

template <int G>
__device__ __forceinline__ float window_weight(const float* __restrict__ T, uint64_t v) {
    const uint32_t vh = static_cast<uint32_t>(v >> 32), vl = static_cast<uint32_t>(v);
    float w = 0.f;
#pragma unroll
    for (int g = 0; g < G; ++g) {
        const uint32_t q = g < 8 ? (vh >> (28 - 4 * g)) & 15u : (vl >> (60 - 4 * g)) & 15u;
        w += T[g * 16 + q];
    }
    return w;
}

// adds z to the accumulator of the symbol that window v shows at this lane's column
__device__ __forceinline__ void accumulate_column(uint64_t v, float z, int colshift, float acc[4]) {
    const unsigned r = static_cast<unsigned>(v >> colshift) & 3u;
    acc[0] += r == 0 ? z : 0.f;
    acc[1] += r == 1 ? z : 0.f;
    acc[2] += r == 2 ? z : 0.f;
    acc[3] += r == 3 ? z : 0.f;
}

template <int G>
__global__ void em_refine_kernel(const EmParams p) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int nwarps = blockDim.x >> 5;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int l = p.l, t = p.t;

    // ---- shared memory carve-up
    float* th = reinterpret_cast<float*>(smem_raw);               // [32][4]
    float* T = th + 128;                                          // [16][16]
    float* part = T + 256;                                        // [nwarps][32][4]
    float* rawm = part + nwarps * 128;                            // [32][4]
    double* llpart = reinterpret_cast<double*>(rawm + 128);       // [nwarps]
    double* dscal = llpart + nwarps;                              // [0] prev_ll  [1..4] log bg
    uint64_t* cand_v = reinterpret_cast<uint64_t*>(dscal + 8);    // [nwarps][kCandCap]
    float* cand_w = reinterpret_cast<float*>(cand_v + nwarps * kCandCap);  // [nwarps][kCandCap]
    int* prof = reinterpret_cast<int*>(cand_w + nwarps * kCandCap);        // [32][4]
    int* iscal = prof + 128;                                      // [0] stop flag [1] score [2] bad
    unsigned long long* cons_bits = reinterpret_cast<unsigned long long*>(iscal + 4);

    uint64_t* my_v = cand_v + warp * kCandCap;
    float* my_w = cand_w + warp * kCandCap;
    const int colshift = 62 - 2 * lane;  // this lane's column in a top-aligned window (lane < l)

    const unsigned int n_work = p.n_work_dev ? *p.n_work_dev : p.n_work;
    for (unsigned int wi = blockIdx.x; wi < n_work; wi += gridDim.x) {
        const WorkDesc wd = p.work[wi];
        __syncthreads();  // previous bucket fully retired before smem reuse

        // ---- init_model (refine.hpp:90-127), pseudocount 0: integer symbol counts of the members
        for (int i = threadIdx.x; i < 128; i += blockDim.x) {
            prof[i] = 0;
            rawm[i] = 0.f;
        }
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
        if (threadIdx.x < 4 * (l + 1)) {
            const int c = threadIdx.x >> 2, r = threadIdx.x & 3;
            th[threadIdx.x] = c == 0 ? static_cast<float>(p.tot_sym[r] / p.tot_bases)
                                     : static_cast<float>(prof[(c - 1) * 4 + r]) / static_cast<float>(wd.count);
        }
        __syncthreads();

        // Sweeps: each EM iteration is one E+M sweep over the sequences; once the iteration budget is
        // spent or the likelihood gain drops below tol, one more sweep does the final E-step
        // (per-sequence argmax) of refine.hpp:306-318.
        int iterations = 0;
        bool final_pass = false;
        for (;;) {
            // ---- log tables for the current theta (refine.hpp:155-161)
            for (int e = threadIdx.x; e < 16 * G; e += blockDim.x) {
                const int g = e >> 4, q = e & 15;
                const int a = q >> 2, b = q & 3;
                const int c0 = 2 * g, c1 = 2 * g + 1;
                float v = 0.f;
                if (c0 < l) v = logf(fmaxf(th[(c0 + 1) * 4 + a], 1e-9f)) - logf(fmaxf(th[a], 1e-9f));
                if (c1 < l) v += logf(fmaxf(th[(c1 + 1) * 4 + b], 1e-9f)) - logf(fmaxf(th[b], 1e-9f));
                T[e] = v;
            }
            if (threadIdx.x < 4) dscal[1 + threadIdx.x] = log(fmax(static_cast<double>(th[threadIdx.x]), 1e-9));
            if (final_pass) {
                for (int i = threadIdx.x; i < 128; i += blockDim.x) prof[i] = 0;
                if (threadIdx.x == 0) {
                    iscal[1] = 0;
                    *cons_bits = 0ULL;
                }
            }
            __syncthreads();

            float acc[4] = {0.f, 0.f, 0.f, 0.f};
            double ll_warp = 0.0;
            for (int i = warp; i < t; i += nwarps) {
                const uint64_t* __restrict__ wp = p.words + p.word_off[i];
                const int n = p.seq_len[i];
                const int W = n - l + 1;
                const int chunks = (W + 31) >> 5;
                float M = -INFINITY, ssum = 0.f;
                int ncand = 0;
                bool overflow = false;
                float best_w = -INFINITY;
                int best_j = 0;
                uint64_t hi = wp[0];
                for (int c = 0; c < chunks; ++c) {
                    const uint64_t lo = wp[c + 1];
                    const int j = (c << 5) + lane;
                    const uint64_t v = window_bits(hi, lo, 2 * lane);
                    hi = lo;
                    const float w = j < W ? window_weight<G>(T, v) : -INFINITY;
                    if (final_pass) {
                        if (w > best_w) {  // strict: the lane keeps its earliest maximum
                            best_w = w;
                            best_j = j;
                        }
                        continue;
                    }
                    const float cm = warp_max_f(w);
                    if (cm > M) {  // warp-uniform
                        ssum *= __expf(M - cm);
                        M = cm;
                    }
                    ssum += __expf(w - M);
                    const bool keep = w >= M + p.log_z_eps;  // superset of the final z >= eps test
                    const unsigned ball = __ballot_sync(0xffffffffu, keep);
                    if (ball && !overflow) {
                        const int cnt = __popc(ball);
                        if (ncand + cnt > kCandCap) {
                            overflow = true;
                        } else {
                            if (keep) {
                                const int slot = ncand + __popc(ball & ((1u << lane) - 1u));
                                my_v[slot] = v;
                                my_w[slot] = w;
                            }
                            ncand += cnt;
                        }
                    }
                }
                if (final_pass) {
                    // per-sequence argmax, ties to the smallest offset (refine.hpp:311-316)
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) {
                        const float ow = __shfl_xor_sync(0xffffffffu, best_w, o);
                        const int oj = __shfl_xor_sync(0xffffffffu, best_j, o);
                        if (ow > best_w || (ow == best_w && oj < best_j)) {
                            best_w = ow;
                            best_j = oj;
                        }
                    }
                    if (!(best_w > -INFINITY) || !(best_w < INFINITY)) iscal[2] = 1;
                    if (p.out_pos && lane == 0) p.out_pos[static_cast<int64_t>(wi) * t + i] = best_j + 1;
                    if (lane < l) {
                        const uint64_t v = load_window(wp, best_j);
                        atomicAdd(&prof[lane * 4 + (static_cast<unsigned>(v >> colshift) & 3u)], 1);
                    }
                    continue;
                }
                const float total = warp_sum_f(ssum);
                if (!(M > -INFINITY) || !(M < INFINITY) || !(total > 0.f)) iscal[2] = 1;
                const float inv_total = 1.f / total;
                // log P(S_i) = sum_r cnt[r] log bg[r] - log W + max + log sum   (refine.hpp:200)
                {
                    const unsigned int* sc = p.seq_sym + i * 4;
                    const double log_base = sc[0] * dscal[1] + sc[1] * dscal[2] + sc[2] * dscal[3] + sc[3] * dscal[4];
                    ll_warp += log_base - p.seq_logw[i] + static_cast<double>(M) +
                               log(static_cast<double>(total));
                }
                __syncwarp();
                if (!overflow) {
                    for (int e = lane; e < ncand; e += 32) {
                        const float z = expf(my_w[e] - M) * inv_total;
                        my_w[e] = (z >= p.z_eps && z > 0.f) ? z : 0.f;
                    }
                    __syncwarp();
                    if (lane < l) {
                        for (int e = 0; e < ncand; ++e) accumulate_column(my_v[e], my_w[e], colshift, acc);
                    }
                    __syncwarp();
                } else {
                    // too many candidates for the list: second sweep with the final max and sum,
                    // flushing the list whenever it fills (exact same predicate and weights)
                    int nl = 0;
                    hi = wp[0];
                    for (int c = 0; c < chunks; ++c) {
                        const uint64_t lo = wp[c + 1];
                        const int j = (c << 5) + lane;
                        const uint64_t v = window_bits(hi, lo, 2 * lane);
                        hi = lo;
                        float z = 0.f;
                        if (j < W) z = expf(window_weight<G>(T, v) - M) * inv_total;
                        const bool keep = z >= p.z_eps && z > 0.f;
                        const unsigned ball = __ballot_sync(0xffffffffu, keep);
                        if (keep) {
                            const int slot = nl + __popc(ball & ((1u << lane) - 1u));
                            my_v[slot] = v;
                            my_w[slot] = z;
                        }
                        nl += __popc(ball);
                        __syncwarp();
                        if (nl > kCandCap - 32 || c == chunks - 1) {
                            if (lane < l) {
                                for (int e = 0; e < nl; ++e) accumulate_column(my_v[e], my_w[e], colshift, acc);
                            }
                            nl = 0;
                            __syncwarp();
                        }
                    }
                }
            }

            if (final_pass) break;

            // ---- M-step (refine.hpp:227-269): deterministic fixed-order reduction over warps
            part[(warp * 32 + lane) * 4 + 0] = acc[0];
            part[(warp * 32 + lane) * 4 + 1] = acc[1];
            part[(warp * 32 + lane) * 4 + 2] = acc[2];
            part[(warp * 32 + lane) * 4 + 3] = acc[3];
            if (lane == 0) llpart[warp] = ll_warp;
            __syncthreads();
            if (threadIdx.x < 4 * l) {
                float sum = 0.f;
                for (int w = 0; w < nwarps; ++w) sum += part[w * 128 + threadIdx.x];
                rawm[threadIdx.x] = sum;  // [c][r]
            }
            __syncthreads();
            if (threadIdx.x <= l) {
                float raw[4];
                if (threadIdx.x < l) {
#pragma unroll
                    for (int r = 0; r < 4; ++r) raw[r] = rawm[threadIdx.x * 4 + r];
                } else {
                    // background = symbol totals - expected motif counts, clamped at 0 (refine.hpp:241-253)
#pragma unroll
                    for (int r = 0; r < 4; ++r) {
                        double b = p.tot_sym[r];
                        for (int c = 0; c < l; ++c) b -= static_cast<double>(rawm[c * 4 + r]);
                        raw[r] = static_cast<float>(fmax(b, 0.0));
                    }
                }
                // write_column (refine.hpp:256-269): normalise, floor at 1e-9, renormalise
                const float sum = raw[0] + raw[1] + raw[2] + raw[3];
                float fs = 0.f;
#pragma unroll
                for (int r = 0; r < 4; ++r) {
                    raw[r] = sum > 0.f ? fmaxf(raw[r] / sum, 1e-9f) : 0.25f;
                    fs += raw[r];
                }
                const int col = threadIdx.x < l ? threadIdx.x + 1 : 0;
#pragma unroll
                for (int r = 0; r < 4; ++r) th[col * 4 + r] = raw[r] / fs;
            }
            ++iterations;
            if (threadIdx.x == 0) {
                double ll = 0.0;
                for (int w = 0; w < nwarps; ++w) ll += llpart[w];
                if (p.out_ll) p.out_ll[static_cast<int64_t>(wi) * p.max_iters + (iterations - 1)] = ll;
                // refine.hpp:296-304: ll is the likelihood of the model ENTERING this iteration; stop
                // after iteration it >= 2 when its gain over the previous one is below tol
                iscal[0] = (iterations >= 2 && ll - dscal[0] < p.tol) ? 1 : 0;
                dscal[0] = ll;
            }
            __syncthreads();
            final_pass = iscal[0] != 0 || iterations >= p.max_iters;
        }

        // ---- score / consensus over the argmax rows (scoring.hpp:84-126), expectation (refine.hpp:130-136)
        __syncthreads();
        if (threadIdx.x < l) {
            const int* pc = prof + threadIdx.x * 4;
            int best = 0;
            for (int r = 1; r < 4; ++r) {
                if (pc[r] > pc[best]) best = r;  // ties go to the lowest rank
            }
            atomicAdd(&iscal[1], pc[best]);
            atomicOr(cons_bits, static_cast<unsigned long long>(best) << (62 - 2 * threadIdx.x));
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            double ex = 0.0;
            for (int c = 1; c <= l; ++c) {
                const float* tc = th + c * 4;
                ex += static_cast<double>(fmaxf(fmaxf(tc[0], tc[1]), fmaxf(tc[2], tc[3])));
            }
            p.out_score[wi] = iscal[1];
            p.out_iters[wi] = iterations;
            p.out_exp[wi] = ex;
            p.out_cons[wi] = *cons_bits;
            atomicAdd(p.iter_total, static_cast<unsigned long long>(iterations + 1));
            if (iscal[2]) atomicExch(p.error_flag, 1u);
        }
        if (p.out_theta && threadIdx.x < 4 * (l + 1)) {
            const int c = threadIdx.x >> 2, r = threadIdx.x & 3;
            p.out_theta[static_cast<int64_t>(wi) * 4 * (l + 1) + r * (l + 1) + c] = static_cast<double>(th[threadIdx.x]);
        }
    }
}

// ---------------------------------------------------------------------------------------------
// per-trial best candidate under candidate_improves (driver.hpp:127-135): higher score, then
// higher expectation, then smaller key.  One warp per trial.
// ---------------------------------------------------------------------------------------------
__device__ __forceinline__ bool better(int sa, double ea, uint64_t ka, int sb, double eb, uint64_t kb) {
    if (sa != sb) return sa > sb;
    if (ea != eb) return ea > eb;
    return ka < kb;
}

// ---------------------------------------------------------------------------------------------
// XOR/popcount Hamming scan: warp per sequence, lane-strided windows.  Two 2-bit digits differ
// iff (x | x>>1) & 01 is set in their XOR x.
// ---------------------------------------------------------------------------------------------
__global__ void hamming_scan_kernel(const uint64_t* __restrict__ words, const int64_t* __restrict__ word_off,
                                    const int32_t* __restrict__ seq_len, int t, int l, uint64_t cand,
                                    int32_t* __restrict__ per_seq_min) {
    const int lane = threadIdx.x & 31;
    const int warps = (gridDim.x * blockDim.x) >> 5;
    const uint64_t digit_mask = (0x5555555555555555ULL >> (64 - 2 * l)) << (64 - 2 * l);
    for (int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < t; i += warps) {
        const uint64_t* wp = words + word_off[i];
        const int W = seq_len[i] - l + 1;
        int best = 64;
        for (int j = lane; j < W; j += 32) {
            const uint64_t xr = load_window(wp, j) ^ cand;
            best = min(best, __popcll((xr | (xr >> 1)) & digit_mask));
        }
        best = __reduce_min_sync(0xffffffffu, best);
        if (lane == 0) per_seq_min[i] = best;
    }
}

// ---------------------------------------------------------------------------------------------
// median_string (oracle.hpp:120-149): exhaustive search over the 4^l candidates for the first minimiser of
// TotalDistance(v) = sum_i min_j hamming(v, S_ij) (oracle.hpp:101-115).  Thread = kMedianCands candidate codes
// (a code is the l-mer itself: first base most significant, kmer.hpp:57-69); the windows of one sequence at a
// time are expanded into shared memory as top-aligned 32-bit l-mers (l <= 16) and every thread scans them with
// XOR/popcount.  Result: min over candidates of (distance << 32 | code), i.e. the smallest code among the
// minimisers -- the reference's "first minimiser in ascending code order".
// ---------------------------------------------------------------------------------------------
constexpr int kMedianThreads = 256;
constexpr int kMedianCands = 4;
constexpr int kMedianChunk = 4096;  // windows staged per round (16 KB)

__global__ void __launch_bounds__(kMedianThreads)
median_string_kernel(const uint64_t* __restrict__ words, const int64_t* __restrict__ word_off,
                     const int32_t* __restrict__ seq_len, int t, int l, uint64_t n_cand,
                     unsigned long long* __restrict__ best) {
    __shared__ uint32_t win[kMedianChunk];
    const uint32_t digit_mask = (0x55555555u >> (32 - 2 * l)) << (32 - 2 * l);
    const int up = 32 - 2 * l;
    const uint64_t per_tile = static_cast<uint64_t>(kMedianThreads) * kMedianCands;
    for (uint64_t tile = blockIdx.x; tile * per_tile < n_cand; tile += gridDim.x) {
        uint32_t cand[kMedianCands];
        int total[kMedianCands];
#pragma unroll
        for (int k = 0; k < kMedianCands; ++k) {
            const uint64_t code = tile * per_tile + static_cast<uint64_t>(k) * kMedianThreads + threadIdx.x;
            cand[k] = static_cast<uint32_t>(code) << up;  // codes past n_cand are computed and discarded
            total[k] = 0;
        }
        for (int i = 0; i < t; ++i) {
            const uint64_t* wp = words + word_off[i];
            const int W = seq_len[i] - l + 1;
            int seq_best[kMedianCands];
#pragma unroll
            for (int k = 0; k < kMedianCands; ++k) seq_best[k] = l + 1;
            for (int start = 0; start < W; start += kMedianChunk) {
                const int cnt = min(kMedianChunk, W - start);
                __syncthreads();
                for (int j = threadIdx.x; j < cnt; j += kMedianThreads) win[j] = static_cast<uint32_t>(load_window(wp, start + j) >> 32);
                __syncthreads();
#pragma unroll 4
                for (int j = 0; j < cnt; ++j) {
                    const uint32_t v = win[j];  // warp-uniform address: one broadcast load
#pragma unroll
                    for (int k = 0; k < kMedianCands; ++k) {
                        const uint32_t xr = v ^ cand[k];
                        seq_best[k] = min(seq_best[k], __popc((xr | (xr >> 1)) & digit_mask));
                    }
                }
            }
#pragma unroll
            for (int k = 0; k < kMedianCands; ++k) total[k] += seq_best[k];
        }
        unsigned long long mine = ~0ULL;
#pragma unroll
        for (int k = 0; k < kMedianCands; ++k) {
            const uint64_t code = tile * per_tile + static_cast<uint64_t>(k) * kMedianThreads + threadIdx.x;
            if (code < n_cand) mine = min(mine, (static_cast<unsigned long long>(total[k]) << 32) | code);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) mine = min(mine, __shfl_xor_sync(0xffffffffu, mine, o));
        if ((threadIdx.x & 31) == 0 && mine != ~0ULL) atomicMin(best, mine);
    }
}

// profile score + consensus of one start vector (0-based starts), single CTA
__global__ void score_kernel(const uint64_t* __restrict__ words, const int64_t* __restrict__ word_off, int t, int l,
                             const int32_t* __restrict__ starts0, int32_t* __restrict__ out_score,
                             uint64_t* __restrict__ out_cons) {
    __shared__ int prof[128];
    __shared__ int score;
    __shared__ unsigned long long cons;
    for (int i = threadIdx.x; i < 128; i += blockDim.x) prof[i] = 0;
    if (threadIdx.x == 0) {
        score = 0;
        cons = 0ULL;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < t; i += blockDim.x) {
        const uint64_t v = load_window(words + word_off[i], starts0[i]);
        for (int c = 0; c < l; ++c) atomicAdd(&prof[c * 4 + (static_cast<unsigned>(v >> (62 - 2 * c)) & 3u)], 1);
    }
    __syncthreads();
    if (threadIdx.x < l) {
        const int* pc = prof + threadIdx.x * 4;
        int best = 0;
        for (int r = 1; r < 4; ++r) {
            if (pc[r] > pc[best]) best = r;
        }
        atomicAdd(&score, pc[best]);
        atomicOr(&cons, static_cast<unsigned long long>(best) << (62 - 2 * threadIdx.x));
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        *out_score = score;
        *out_cons = cons;
    }
}

// (x - size) keys for ordering enriched records by size descending with the stable sorter
__global__ void size_keys_kernel(const unsigned int* __restrict__ rec_size, const unsigned int* __restrict__ n_rec,
                                 int64_t cap_e, unsigned int x, int n_trials, unsigned int* __restrict__ keys) {
    for (int tr = blockIdx.y; tr < n_trials; tr += gridDim.y) {
        const unsigned int ne = min(n_rec[tr], static_cast<unsigned int>(cap_e));
        for (unsigned int e = blockIdx.x * blockDim.x + threadIdx.x; e < ne; e += gridDim.x * blockDim.x) {
            const int64_t o = static_cast<int64_t>(tr) * cap_e + e;
            keys[o] = x - rec_size[o];
        }
    }
}

}  // namespace k
}  // namespace pm
