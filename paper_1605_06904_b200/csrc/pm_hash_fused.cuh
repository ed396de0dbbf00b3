// pm_hash_fused.cuh — hash_trial + enriched_buckets of one trial in ONE CTA (projection.hpp:319-390) for the
// trial loop of run(): the shared-memory-privatised histogram alternative that north_star names.
//
// Applies when the dense table fits shared memory (4^k <= 65,536, the reference's own dense_table_cap) and the
// set is small (x < 65,536 l-mers, packed words <= 16 KB): every t=20 configuration.  Per trial:
//   pass 1   every l-mer -> projected key -> shared-memory counter (16-bit counters, two per word)
//   scan     keys in ascending order: buckets with count >= s get a record (key, first member slot, size)
//            by a block-wide exclusive scan, i.e. the compaction is in key order like the sorted path
//   pass 2   l-mers of enriched buckets take a slot of their bucket (shared-memory cursor)
//   sort     each bucket's few members are put in ascending l-mer order ((seq, offset) order, projection.hpp:275-277)
// The packed words are staged once per CTA with a TMA bulk copy and stay resident for all its trials.
// Output is what the sort path produces for run(): records in key order and, for their buckets, the member
// lists at the same offsets convention (trial * x + start).  Algorithmic bytes per trial: ceil(t n / 4) read
// (once per CTA, from L2) + 8 bytes per enriched member and 16 per record written; nothing else touches HBM.
#pragma once
#include "pm_em_smem.cuh"

namespace pm {
namespace k {

constexpr int kFusedThreads = 512;
constexpr int kFusedBigBucket = 96;  // buckets above this size are ordered cooperatively by rank counting

struct FusedHashParams {
    const uint64_t* words;
    const int64_t* word_off;
    const int64_t* win_off;  // [t+1] first flat l-mer index of each sequence
    int t, keybits;
    int x;        // l-mers per trial (< 65,536)
    int n_words;  // packed words of the whole set
    int thr;      // bucket threshold s
    int cap_e;    // record capacity per trial (x / s)
    int plan_base, n_trials;
    unsigned int* members;  // [trial][x] flat l-mer indices, bucket by bucket
    uint64_t* rec_key;      // [trial][cap_e]
    unsigned int* rec_start;
    unsigned int* rec_size;
    unsigned int* n_rec;    // [trial]
};

__device__ __forceinline__ unsigned int project_prog(const PlanProg& pp, uint64_t v) {
    uint64_t key = 0;
    const int nruns = pp.nruns;
    for (int r = 0; r < nruns; ++r) {
        const int nb = pp.nbits[r];
        key = (key << nb) | ((v >> pp.rshift[r]) & ((1ULL << nb) - 1ULL));
    }
    return static_cast<unsigned int>(key);
}

__global__ void __launch_bounds__(kFusedThreads)
hash_bucket_fused_kernel(const FusedHashParams p) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int n_keys = 1 << p.keybits;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr int kWarps = kFusedThreads / 32;
    // ---- carve-up (mirrored by fused_hash_smem_bytes)
    uint64_t* wstage = reinterpret_cast<uint64_t*>(smem_raw);                              // [n_words]
    unsigned int* cnt = reinterpret_cast<unsigned int*>(wstage + p.n_words);               // [n_keys / 2] 2 x u16
    unsigned int* enr = cnt + (n_keys >> 1);                                               // [n_keys / 32] enriched bits
    unsigned int* rec_s = enr + max(n_keys >> 5, 1);                                       // [cap_e] base | size << 16
    int* seq_first = reinterpret_cast<int*>(rec_s + p.cap_e);                              // [t + 1] win_off
    int* seq_word = seq_first + p.t + 1;                                                   // [t] word offset
    unsigned int* wsum = reinterpret_cast<unsigned int*>(seq_word + p.t);                  // [2][kWarps] scan partials
    unsigned int* scal = wsum + 2 * kWarps;                                                // [0] records [1] members
    uint16_t* mem_s = reinterpret_cast<uint16_t*>(scal + 2);                               // [x]
    unsigned long long* mbar = reinterpret_cast<unsigned long long*>(
        smem_raw + ((static_cast<unsigned int>(reinterpret_cast<unsigned char*>(mem_s + p.x) - smem_raw) + 7u) & ~7u));

    if (tid == 0) {
        mbar_init(mbar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        mbar_expect_tx(mbar, static_cast<unsigned>(p.n_words) * 8u);
        tma_load_1d(wstage, p.words, static_cast<unsigned>(p.n_words) * 8u, mbar);
    }
    for (int i = tid; i <= p.t; i += kFusedThreads) seq_first[i] = static_cast<int>(p.win_off[i]);
    for (int i = tid; i < p.t; i += kFusedThreads) seq_word[i] = static_cast<int>(p.word_off[i] - p.word_off[0]);
    __syncthreads();
    mbar_wait(mbar, 0);

    for (int tr = blockIdx.x; tr < p.n_trials; tr += gridDim.x) {
        const PlanProg& pp = c_plans[tr];
        const int64_t trial = p.plan_base + tr;
        for (int i = tid; i < (n_keys >> 1); i += kFusedThreads) cnt[i] = 0u;
        for (int i = tid; i < max(n_keys >> 5, 1); i += kFusedThreads) enr[i] = 0u;
        __syncthreads();

        // ---- pass 1: histogram of the projected keys
        {
            int i = 0;
            for (int f = tid; f < p.x; f += kFusedThreads) {
                while (f >= seq_first[i + 1]) ++i;
                const unsigned int key = project_prog(pp, load_window(wstage + seq_word[i], f - seq_first[i]));
                atomicAdd(&cnt[key >> 1], 1u << ((key & 1u) * 16u));
            }
        }
        __syncthreads();

        // ---- enriched keys in ascending order: thread `tid` owns keys [tid*per, (tid+1)*per)
        const int per = (n_keys + kFusedThreads - 1) / kFusedThreads;
        const int k_lo = min(tid * per, n_keys), k_hi = min(k_lo + per, n_keys);
        unsigned int my_rec = 0, my_mem = 0;
        for (int key = k_lo; key < k_hi; ++key) {
            const unsigned int c = (cnt[key >> 1] >> ((key & 1) * 16)) & 0xFFFFu;
            if (c >= static_cast<unsigned int>(p.thr)) {
                ++my_rec;
                my_mem += c;
            }
        }
        // block-wide exclusive scans of (records, members)
        unsigned int inc_rec = my_rec, inc_mem = my_mem;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned int a = __shfl_up_sync(0xffffffffu, inc_rec, o), b = __shfl_up_sync(0xffffffffu, inc_mem, o);
            if (lane >= o) {
                inc_rec += a;
                inc_mem += b;
            }
        }
        if (lane == 31) {
            wsum[warp] = inc_rec;
            wsum[kWarps + warp] = inc_mem;
        }
        __syncthreads();
        unsigned int base_rec = inc_rec - my_rec, base_mem = inc_mem - my_mem;
        for (int w = 0; w < warp; ++w) {
            base_rec += wsum[w];
            base_mem += wsum[kWarps + w];
        }
        if (tid == kFusedThreads - 1) {
            scal[0] = base_rec + my_rec;
            scal[1] = base_mem + my_mem;
        }
        // records (global + shared copy) and the slot cursor of every enriched key
        for (int key = k_lo; key < k_hi; ++key) {
            const unsigned int sh = (key & 1) * 16;
            const unsigned int c = (cnt[key >> 1] >> sh) & 0xFFFFu;
            if (c >= static_cast<unsigned int>(p.thr)) {
                const int64_t o = trial * p.cap_e + base_rec;
                p.rec_key[o] = static_cast<uint64_t>(key);
                p.rec_start[o] = base_mem;
                p.rec_size[o] = c;
                rec_s[base_rec] = base_mem | (c << 16);
                // count -> slot cursor, touching only this key's half of the word (the other half may belong to
                // another thread when there are fewer keys than threads)
                atomicAnd(&cnt[key >> 1], ~(0xFFFFu << sh));
                atomicOr(&cnt[key >> 1], base_mem << sh);
                atomicOr(&enr[key >> 5], 1u << (key & 31));
                ++base_rec;
                base_mem += c;
            }
        }
        __syncthreads();
        const unsigned int n_rec = scal[0], n_mem = scal[1];

        // ---- pass 2: members of enriched buckets take a slot of their bucket
        {
            int i = 0;
            for (int f = tid; f < p.x; f += kFusedThreads) {
                while (f >= seq_first[i + 1]) ++i;
                const unsigned int key = project_prog(pp, load_window(wstage + seq_word[i], f - seq_first[i]));
                if ((enr[key >> 5] >> (key & 31)) & 1u) {
                    const unsigned int sh = (key & 1u) * 16u;
                    const unsigned int old = atomicAdd(&cnt[key >> 1], 1u << sh);
                    // the cursor of the last bucket may wrap past 0xFFFF only when n_mem == 65,536, excluded by x < 65,536
                    mem_s[(old >> sh) & 0xFFFFu] = static_cast<uint16_t>(f);
                }
            }
        }
        __syncthreads();

        // ---- ascending l-mer order inside each bucket
        for (unsigned int r = tid; r < n_rec; r += kFusedThreads) {
            const unsigned int base = rec_s[r] & 0xFFFFu, size = rec_s[r] >> 16;
            if (size > kFusedBigBucket) continue;
            uint16_t* m = mem_s + base;
            for (unsigned int a = 1; a < size; ++a) {  // insertion sort: sizes are a handful
                const uint16_t v = m[a];
                int b = static_cast<int>(a) - 1;
                while (b >= 0 && m[b] > v) {
                    m[b + 1] = m[b];
                    --b;
                }
                m[b + 1] = v;
            }
        }
        __syncthreads();
        // big buckets (degenerate inputs): every thread ranks a share of the members, staged through global memory
        for (unsigned int r = 0; r < n_rec; ++r) {
            const unsigned int base = rec_s[r] & 0xFFFFu, size = rec_s[r] >> 16;
            if (size <= kFusedBigBucket) continue;  // block-uniform
            unsigned int* out = p.members + trial * p.x + base;
            for (unsigned int a = tid; a < size; a += kFusedThreads) {
                const uint16_t v = mem_s[base + a];
                unsigned int rank = 0;
                for (unsigned int b = 0; b < size; ++b) rank += mem_s[base + b] < v ? 1u : 0u;
                out[rank] = v;  // members are distinct l-mer indices: ranks are a permutation
            }
            __syncthreads();
            for (unsigned int a = tid; a < size; a += kFusedThreads) mem_s[base + a] = static_cast<uint16_t>(out[a]);
            __syncthreads();
        }
        {
            unsigned int* out = p.members + trial * p.x;
            for (unsigned int a = tid; a < n_mem; a += kFusedThreads) out[a] = mem_s[a];
        }
        if (tid == 0) p.n_rec[trial] = n_rec;
        __syncthreads();
    }
}

}  // namespace k
}  // namespace pm
