// pm_capi.cu — device context and the C-ABI entry points of include/pm_b200.h.
//
// Host C++ drives hand-written sm_100a kernels (pm_kernels.cuh) on one CUDA stream.  Nothing here
// computes any part of the path on the CPU: the host samples projection plans (the reference's
// PRNG stream, pm_host.cpp), turns them into constant-memory extraction programs, launches the
// kernels and scans the per-trial summaries in ascending trial order exactly like the
// reduction of driver.hpp:195-208.
#include <algorithm>
#if defined(__SSE2__)
#include <emmintrin.h>
#endif
#include <chrono>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <future>
#include <limits>
#include <map>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include <cuda_runtime.h>

#include "pm_internal.hpp"
#include "pm_kernels.cuh"
#include "pm_em_smem.cuh"
#include "pm_em_pair.cuh"
#include "pm_em_tc.cuh"
#include "pm_em_f64.cuh"
#include "pm_planted.cuh"
#include "pm_hash_fused.cuh"
#include "pm_hash_count.cuh"
#include "pm_plans.cuh"

using namespace pm;

namespace {

#define PM_CUDA(call)                                                                                  \
    do {                                                                                               \
        const cudaError_t e_ = (call);                                                                 \
        if (e_ != cudaSuccess) {                                                                       \
            return set_error(e_ == cudaErrorMemoryAllocation ? PM_ERR_OUT_OF_MEMORY : PM_ERR_CUDA,     \
                             std::string(#call) + ": " + cudaGetErrorString(e_));                      \
        }                                                                                              \
    } while (0)

#define PM_TRY(call)                  \
    do {                              \
        const int rc_ = (call);       \
        if (rc_ != PM_OK) return rc_; \
    } while (0)

// grow-only device buffer
struct DevBuf {
    void* p = nullptr;
    size_t cap = 0;
};

enum Slot {
    S_KEYS_A, S_KEYS_B, S_IDX_A, S_IDX_B, S_COUNTS, S_REC_KEY, S_REC_START, S_REC_SIZE, S_NREC, S_WORK_OFF,
    S_WORK, S_OUT_SCORE, S_OUT_ITERS, S_OUT_EXP, S_OUT_CONS, S_OUT_POS, S_OUT_THETA, S_OUT_LL, S_BEST, S_TB,
    S_SCAL, S_MEMBERS, S_MPREV, S_DIGIT_TOT, S_ETILES, S_TMP_A, S_TMP_B, S_TMP_C, S_TMP_D, S_ASCII, S_OFFS,
    S_TC_BLOCKS, S_TC_FLAG, S_TC_WORK, S_TC_MAP, S_F64_Z, S_F64_FLAG, S_F64_WORK, S_F64_MAP, S_THETA_IN, S_NCLOSE, S_POS_BEST, S_HAM, S_PLANS, S_PLAN_KEPT,
    // the FP64 path has its own scratch: run() calls it while a batch's buffers are still live
    S_DRAWS, S_PLANT_OUT, S_X_MEMBERS, S_X_WORK, S_X_SCAL, S_X_SCORE, S_X_ITERS, S_X_EXP, S_X_CONS, S_X_POS, S_X_THETA, S_X_LL, S_X_THETA_IN, S_COUNT_
};

}  // namespace

struct pm_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    int sm_count = 148;
    int64_t launches = 0;
    // sequence set
    int t = 0;
    std::vector<int64_t> offs, word_off;
    std::vector<int32_t> seq_len;
    int64_t total_bases = 0, total_words = 0;
    uint64_t* d_words = nullptr;
    int64_t* d_word_off = nullptr;
    int32_t* d_seq_len = nullptr;
    unsigned int* d_seq_sym = nullptr;
    unsigned long long* d_tot_sym = nullptr;  // [0..3] symbol totals, [4] first bad byte
    unsigned long long tot_sym[4] = {0, 0, 0, 0};
    // pair-class position groups for the shared-memory EM kernel (built once per sequence set)
    uint16_t* d_cls_entries = nullptr;
    int* d_cls_group_off = nullptr;
    int* d_seq_zoff = nullptr;
    k::TileDesc* d_tiles = nullptr;
    int n_tiles = 0;
    int tile_words = 0;    // most packed words any tile needs (TMA stage size)
    int zlen = 0;          // largest tile's z slots; 0 => some sequence does not fit the shared-memory EM kernel
    int total_groups = 0;
    double group_fill = 0.0;  // live entries / slots of the class-gather rows
    int em_cfg_l = -1, em_cfg_threads = 0, em_cfg_per_sm = 0;  // cached launch setup of the smem EM kernel
    size_t em_cfg_smem = 0;
    int pair_cfg_l = -1, pair_cfg_threads = 0, pair_cfg_per_sm = 0;  // same for the two-bucket kernel
    size_t pair_cfg_smem = 0;
    int32_t max_seq_len = 0;
    int max_tile_seqs = 0;  // most sequences any tile of the class-group index holds
    // tensor-core EM kernel (pm_em_tc.cuh): block list of one sweep for the current (set, l)
    int tc_l = -1, tc_n_blocks = 0, tc_e_positions = 0;
    int64_t tc_g1_flops = 0, tc_g2_flops = 0;  // per tile and pass: GEMM1 with ONE log-odds term, GEMM2 with both P terms
    bool tc_used = false;                      // the last launch_em went through the tensor-core kernel
    std::vector<k::TcBlock> h_tc_blocks;
    k::TcBlock* d_tc_blocks = nullptr;
    int64_t em_exact[6] = {0, 0, 0, 0, 0, 0};  // last refine/run: buckets the tensor-core kernel handed to the pair kernel
                                               // [0] total, then by reason: likelihood gain, range, argmax tie, non-finite;
                                               // [5] buckets the pair kernel handed to the FP64 kernel
    // host staging of the class-group index: lives in the context so the async uploads need no sync of their own
    std::vector<k::TileDesc> h_tiles;
    std::vector<int> h_zoff, h_group_off;
    std::vector<uint16_t> h_entries;
    // The class-group index of a small set is built on a worker thread while the first kernels of the run are already
    // queued (it is only needed by the pair kernel, which follows the tensor-core kernel): see finish_class_groups()
    struct ClsResult {
        int zcap = 0, wcap = 0;
        int64_t live_slots = 0;
        size_t live_rows = 0;
        bool built = false;  // false: a single sequence exceeds the z buffer (streaming kernel)
    };
    // pinned host staging for the per-batch read-back (copies into pageable memory block the host for ~10 us each)
    void* h_pin = nullptr;
    size_t h_pin_cap = 0;
    std::future<ClsResult> cls_job;
    bool cls_pending = false;
    bool cls_hint_small = false;  // known before the build ends: every sequence fits a tile of a small set
    std::string cls_bases;        // the worker's copy of the ASCII input
    std::vector<int64_t> cls_rel, cls_word_off;
    std::vector<double> h_logw;
    // window index space for the current l
    int win_l = 0;
    std::vector<int64_t> win_off;
    int64_t* d_win_off = nullptr;
    double* d_seq_logw = nullptr;
    int64_t x = 0, uniform_w = 0;
    DevBuf buf[S_COUNT_];
    // capacities (bytes) of the per-set device arrays above: reused across pm_ctx_set_sequences calls
    size_t cap_words = 0, cap_word_off = 0, cap_seq_len = 0, cap_seq_sym = 0, cap_tot_sym = 0, cap_win_off = 0,
           cap_seq_logw = 0, cap_cls_entries = 0, cap_cls_group_off = 0, cap_seq_zoff = 0, cap_tiles = 0;
    // measurement: bytes moved by this context and stage timing events (read after a sync)
    int64_t h2d_bytes = 0, d2h_bytes = 0;
    struct StageMark {
        int stage;
        cudaEvent_t a, b;
    };
    std::vector<StageMark> marks;
    std::vector<cudaEvent_t> ev_pool;
};

namespace {

template <typename T>
int get_buf(pm_ctx* c, Slot s, size_t n, T** out) {
    DevBuf& b = c->buf[s];
    const size_t bytes = std::max<size_t>(n, 1) * sizeof(T);
    if (bytes > b.cap) {
        if (b.p != nullptr) {
            PM_CUDA(cudaStreamSynchronize(c->stream));
            PM_CUDA(cudaFree(b.p));
            b.p = nullptr;
            b.cap = 0;
        }
        const size_t want = bytes + bytes / 4;  // a little headroom so growing batches do not thrash
        PM_CUDA(cudaMalloc(&b.p, want));
        b.cap = want;
    }
    *out = static_cast<T*>(b.p);
    return PM_OK;
}

// grow-only allocation of a per-set device array
template <typename T>
int ensure(pm_ctx* c, T** ptr, size_t* cap, size_t bytes) {
    if (*ptr != nullptr && *cap >= bytes) return PM_OK;
    if (*ptr != nullptr) {
        PM_CUDA(cudaStreamSynchronize(c->stream));
        PM_CUDA(cudaFree(*ptr));
        *ptr = nullptr;
        *cap = 0;
    }
    void* p = nullptr;
    PM_CUDA(cudaMalloc(&p, std::max<size_t>(bytes, 16)));
    *ptr = static_cast<T*>(p);
    *cap = std::max<size_t>(bytes, 16);
    return PM_OK;
}

int check_launch(pm_ctx* c, const char* what) {
    ++c->launches;
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return set_error(PM_ERR_CUDA, std::string(what) + " launch: " + cudaGetErrorString(e));
    return PM_OK;
}

// Stage timing without extra synchronisation: events are recorded on the stream and read back by
// collect_stage_times() after the batch's own final cudaStreamSynchronize.
cudaEvent_t take_event(pm_ctx* c) {
    if (!c->ev_pool.empty()) {
        cudaEvent_t e = c->ev_pool.back();
        c->ev_pool.pop_back();
        return e;
    }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
}

struct StageTimer {
    pm_ctx* c;
    bool on;
    int stage;
    cudaEvent_t a = nullptr;
    StageTimer(pm_ctx* ctx, bool enable, int stage_index) : c(ctx), on(enable), stage(stage_index) {
        if (on) {
            a = take_event(c);
            cudaEventRecord(a, c->stream);
        }
    }
    void stop() {
        if (on && a) {
            cudaEvent_t b = take_event(c);
            cudaEventRecord(b, c->stream);
            c->marks.push_back({stage, a, b});
            a = nullptr;
        }
    }
    ~StageTimer() { stop(); }
};

// call only after the stream has been synchronised
void collect_stage_times(pm_ctx* c, double* stage_ms) {
    for (const pm_ctx::StageMark& m : c->marks) {
        float ms = 0.f;
        if (cudaEventElapsedTime(&ms, m.a, m.b) == cudaSuccess) stage_ms[m.stage] += ms;
        c->ev_pool.push_back(m.a);
        c->ev_pool.push_back(m.b);
    }
    c->marks.clear();
}

// pinned host memory of at least `bytes` (grow-only; the previous batch's contents are gone)
int get_pinned(pm_ctx* c, size_t bytes, void** out) {
    if (bytes > c->h_pin_cap) {
        if (c->h_pin != nullptr) {
            PM_CUDA(cudaStreamSynchronize(c->stream));
            PM_CUDA(cudaFreeHost(c->h_pin));
            c->h_pin = nullptr;
            c->h_pin_cap = 0;
        }
        const size_t cap = std::max<size_t>(bytes + bytes / 2, 1 << 16);
        PM_CUDA(cudaHostAlloc(&c->h_pin, cap, cudaHostAllocDefault));
        c->h_pin_cap = cap;
    }
    *out = c->h_pin;
    return PM_OK;
}

int h2d(pm_ctx* c, void* dst, const void* src, size_t bytes) {
    c->h2d_bytes += static_cast<int64_t>(bytes);
    PM_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, c->stream));
    return PM_OK;
}

int d2h(pm_ctx* c, void* dst, const void* src, size_t bytes) {
    c->d2h_bytes += static_cast<int64_t>(bytes);
    PM_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, c->stream));
    return PM_OK;
}

// Index build for the shared-memory EM kernel (pm_em_smem.cuh).  Sequences are split into tiles whose
// responsibilities fit the kernel's z buffer; per tile, the pair class 4*s_p + s_{p+1} of every base
// position is grouped per class into rows of 32 slots with pairwise distinct addresses mod 32, so
// the M-step gather is free of bank conflicts.  A layout table like word_off, not arithmetic of
// the path; it depends on the sequence set only (not on l, the plan or the bucket).
// z slots per tile: one tile up to ~13.5k slots (3 CTAs/SM); above that, balanced tiles of at most ~12.6k slots
// (two tiles for the n=1000 configs: 4 CTAs/SM, measured +5 % over one 84 KB tile)
int64_t class_tile_cap(int64_t total, int t) {
    const int64_t single = k::kZPad + total + 32 * static_cast<int64_t>(t);
    int64_t cap = single;
    if (single > 13500) {
        const int64_t nt = (single + 12599) / 12600;
        cap = single / nt + 700;
    }
    if (const char* env = std::getenv("PM_B200_TILE_SLOTS")) {  // test knob: force small tiles
        const long v = std::atol(env);
        if (v >= 256 && v <= 48000) cap = v;
    }
    return cap;
}

// host part: fills c->h_tiles / h_zoff / h_group_off / h_entries (no CUDA call: may run on a worker thread)
pm_ctx::ClsResult class_groups_cpu(pm_ctx* c, const char* bases, const std::vector<int64_t>& rel,
                                   const std::vector<int64_t>& word_off, int t) {
    pm_ctx::ClsResult res;
    const int64_t total = rel[static_cast<size_t>(t)];
    const int64_t single = k::kZPad + total + 32 * static_cast<int64_t>(t);
    const int64_t cap = class_tile_cap(total, t);
    // Sequences per tile: at most kPairMaxSeqs (the pair kernel keeps a tile's metadata in shared memory), and for
    // multi-tile sets a multiple of the ten warps of a CTA when ten or more fit (warp per sequence: a tile of
    // twelve leaves eight warps idle for half of the E-step).
    int tile_seq_cap = k::kPairMaxSeqs;
    if (single > 13500) {
        const int64_t mean_len = std::max<int64_t>(1, total / t) + 32;
        const int64_t fit = std::max<int64_t>(1, (cap - k::kZPad) / mean_len);
        if (fit >= 10) tile_seq_cap = static_cast<int>(std::min<int64_t>(k::kPairMaxSeqs, fit / 10 * 10));
    }
    auto code = [](char ch) { return (static_cast<unsigned char>(ch) >> 1) & 3; };
    std::vector<k::TileDesc>& tiles = c->h_tiles;
    std::vector<int>& zoff = c->h_zoff;
    std::vector<int>& group_off = c->h_group_off;  // 17 per tile
    std::vector<uint16_t>& entries = c->h_entries;
    tiles.clear();
    zoff.assign(static_cast<size_t>(t), 0);
    group_off.clear();
    entries.clear();
    // per class: residue loads stored twice in a row (load2[q][r] == load2[q][r + 32]) so that the shift search
    // below reads contiguous runs and vectorises
    // (16-bit counters: a tile has fewer than 2^15 positions; eight lanes per SSE2 operation)
    std::vector<int16_t> load2(16 * 64), mine(16 * 32);
    std::vector<uint8_t> qv;  // pair class of every position of the current sequence
    std::vector<uint8_t> tile_q;      // pair class of every position of the current tile, sequence after sequence
    std::vector<uint16_t> tile_slot;  // its z slot
    int64_t live_slots = 0;
    int zcap = 0, wcap = 0;
    int i = 0;
    while (i < t) {
        k::TileDesc tile;
        tile.seq_begin = i;
        tile.group_base = static_cast<int>(entries.size() / 32);
        std::fill(load2.begin(), load2.end(), 0);
        tile_q.clear();
        tile_slot.clear();
        int64_t cursor = k::kZPad;
        while (i < t) {
            const int64_t n = rel[static_cast<size_t>(i) + 1] - rel[static_cast<size_t>(i)];
            if (cursor + 31 + n > cap) break;
            if (i - tile.seq_begin >= tile_seq_cap) break;
            const char* sq = bases + rel[static_cast<size_t>(i)];
            // the slack before this sequence (0..31 slots) is chosen greedily so that, per class, the
            // positions spread evenly over the 32 address residues (rows of a class = its fullest residue)
            std::fill(mine.begin(), mine.end(), 0);
            qv.resize(static_cast<size_t>(n));
            for (int64_t p = 0; p < n; ++p) {
                const int q = 4 * code(sq[p]) + (p + 1 < n ? code(sq[p + 1]) : 0);
                qv[static_cast<size_t>(p)] = static_cast<uint8_t>(q);
                ++mine[static_cast<size_t>(q * 32 + ((cursor + p) & 31))];
            }
            int best_shift = 0;
            int64_t best_cost = -1;
            for (int sh = 0; sh < 32; ++sh) {
                int64_t cost = 0;
                for (int q = 0; q < 16; ++q) {
                    const int16_t* __restrict__ lq = load2.data() + q * 64 + sh;  // lq[r] = load[q][(r + sh) & 31]
                    const int16_t* __restrict__ mq = mine.data() + q * 32;
#if defined(__SSE2__)
                    __m128i mx8 = _mm_setzero_si128();
                    for (int r = 0; r < 32; r += 8) {
                        const __m128i a = _mm_loadu_si128(reinterpret_cast<const __m128i*>(lq + r));
                        const __m128i b = _mm_loadu_si128(reinterpret_cast<const __m128i*>(mq + r));
                        mx8 = _mm_max_epi16(mx8, _mm_add_epi16(a, b));
                    }
                    mx8 = _mm_max_epi16(mx8, _mm_srli_si128(mx8, 8));
                    mx8 = _mm_max_epi16(mx8, _mm_srli_si128(mx8, 4));
                    mx8 = _mm_max_epi16(mx8, _mm_srli_si128(mx8, 2));
                    cost += static_cast<int16_t>(_mm_extract_epi16(mx8, 0));
#else
                    int mx = 0;
                    for (int r = 0; r < 32; ++r) mx = std::max(mx, lq[r] + mq[r]);
                    cost += mx;
#endif
                }
                if (best_cost < 0 || cost < best_cost) {
                    best_cost = cost;
                    best_shift = sh;
                }
            }
            for (int q = 0; q < 16; ++q) {
                for (int r = 0; r < 32; ++r) {
                    const int dst = (r + best_shift) & 31;
                    load2[static_cast<size_t>(q * 64 + dst)] += mine[static_cast<size_t>(q * 32 + r)];
                    load2[static_cast<size_t>(q * 64 + dst + 32)] = load2[static_cast<size_t>(q * 64 + dst)];
                }
            }
            cursor += best_shift;
            zoff[static_cast<size_t>(i)] = static_cast<int>(cursor);
            tile_q.insert(tile_q.end(), qv.begin(), qv.end());
            {
                const size_t at = tile_slot.size();
                tile_slot.resize(at + static_cast<size_t>(n));
                for (int64_t p = 0; p < n; ++p) tile_slot[at + static_cast<size_t>(p)] = static_cast<uint16_t>(cursor + p);
            }
            cursor += n;
            live_slots += n;
            ++i;
        }
        if (i == tile.seq_begin) return res;  // a single sequence exceeds the z buffer: streaming kernel
        tile.seq_end = i;
        tile.zlen = static_cast<int>(cursor);
        tile.word_begin = word_off[static_cast<size_t>(tile.seq_begin)];
        tile.n_words = static_cast<int>(word_off[static_cast<size_t>(tile.seq_end)] - tile.word_begin);
        wcap = std::max(wcap, tile.n_words);
        zcap = std::max(zcap, tile.zlen);
        int row = 0;
        // rows of class q = its fullest residue (load2 holds the per-residue counts of the finished tile); every
        // row starts as dummies (zero slot of the same bank) and positions fill their residue's lane in order
        int first_row[16];
        for (int q = 0; q < 16; ++q) {
            group_off.push_back(row);
            first_row[q] = row;
            int rows = 0;
            for (int r = 0; r < 32; ++r) rows = std::max<int>(rows, load2[static_cast<size_t>(q * 64 + r)]);
            row += rows;
        }
        group_off.push_back(row);
        const size_t base = entries.size();
        entries.resize(base + static_cast<size_t>(row) * 32);
        for (size_t e = base; e < entries.size(); ++e) entries[e] = static_cast<uint16_t>(32 + ((e - base) & 31));
        int16_t placed[16 * 32] = {0};
        for (size_t p = 0; p < tile_q.size(); ++p) {
            const int q = tile_q[p], r = tile_slot[p] & 31;
            const int g = placed[q * 32 + r]++;
            entries[base + (static_cast<size_t>(first_row[q]) + static_cast<size_t>(g)) * 32 + static_cast<size_t>(r)] = tile_slot[p];
        }
        tiles.push_back(tile);
    }
    res.live_rows = entries.size() / 32;
    for (int r = 0; r < 2 * 32; ++r) entries.push_back(static_cast<uint16_t>(32 + (r & 31)));  // rows the gather's prefetch may touch
    res.zcap = zcap;
    res.wcap = wcap;
    res.live_slots = live_slots;
    res.built = true;
    return res;
}

// device part: uploads the tables and publishes the geometry in the context
int class_groups_upload(pm_ctx* c, const pm_ctx::ClsResult& res, int t) {
    if (!res.built) return PM_OK;
    const std::vector<k::TileDesc>& tiles = c->h_tiles;
    PM_TRY(ensure(c, &c->d_cls_entries, &c->cap_cls_entries, sizeof(uint16_t) * std::max<size_t>(c->h_entries.size(), 1)));
    PM_TRY(ensure(c, &c->d_cls_group_off, &c->cap_cls_group_off, sizeof(int) * c->h_group_off.size()));
    PM_TRY(ensure(c, &c->d_seq_zoff, &c->cap_seq_zoff, sizeof(int) * static_cast<size_t>(t)));
    PM_TRY(ensure(c, &c->d_tiles, &c->cap_tiles, sizeof(k::TileDesc) * tiles.size()));
    PM_TRY(h2d(c, c->d_cls_entries, c->h_entries.data(), sizeof(uint16_t) * c->h_entries.size()));
    PM_TRY(h2d(c, c->d_cls_group_off, c->h_group_off.data(), sizeof(int) * c->h_group_off.size()));
    PM_TRY(h2d(c, c->d_seq_zoff, c->h_zoff.data(), sizeof(int) * c->h_zoff.size()));
    PM_TRY(h2d(c, c->d_tiles, tiles.data(), sizeof(k::TileDesc) * tiles.size()));
    // no sync here: the staging vectors belong to the context; the next upload starts with a stream synchronisation
    c->zlen = res.zcap;
    c->max_tile_seqs = 0;
    for (const k::TileDesc& td : tiles) c->max_tile_seqs = std::max(c->max_tile_seqs, td.seq_end - td.seq_begin);
    c->tile_words = res.wcap;
    c->n_tiles = static_cast<int>(tiles.size());
    c->total_groups = static_cast<int>(res.live_rows);
    c->group_fill = res.live_rows == 0 ? 0.0 : static_cast<double>(res.live_slots) / static_cast<double>(res.live_rows * 32);
    return PM_OK;
}

// joins the worker of the last upload, if any, and uploads its tables
int finish_class_groups(pm_ctx* c) {
    if (!c->cls_pending) return PM_OK;
    c->cls_pending = false;
    pm_ctx::ClsResult res;
    try {
        res = c->cls_job.get();
    } catch (const std::exception& e) {
        return set_error(PM_ERR_OUT_OF_MEMORY, std::string("class-group build failed: ") + e.what());
    }
    return class_groups_upload(c, res, static_cast<int>(c->h_zoff.size()));
}

// PM_B200_HOST_TIMING=1: wall-clock marks of the host side of pm_run on stderr (where the GPU may sit idle)
struct HostMarks {
    bool on = std::getenv("PM_B200_HOST_TIMING") != nullptr;
    std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
    std::string line;
    void mark(const char* what) {
        if (!on) return;
        const auto now = std::chrono::steady_clock::now();
        char buf[64];
        std::snprintf(buf, sizeof(buf), " %s %.0fus", what, std::chrono::duration<double, std::micro>(now - t0).count());
        line += buf;
        t0 = now;
    }
    ~HostMarks() {
        if (on && !line.empty()) std::fprintf(stderr, "[pm host]%s\n", line.c_str());
    }
};
thread_local HostMarks* g_marks = nullptr;
void host_mark(const char* what) {
    if (g_marks) g_marks->mark(what);
}

int need_sequences(const pm_ctx* c) {
    if (c == nullptr) return set_error(PM_ERR_INVALID_PARAMS, "null context");
    if (c->t < 1) return set_error(PM_ERR_INVALID_PARAMS, "no sequence set loaded: call pm_ctx_set_sequences first");
    return PM_OK;
}

// (seq, offset) index space for motif length l (sequence.hpp:103-132)
int prepare_windows(pm_ctx* c, int l) {
    PM_CUDA(cudaSetDevice(c->device));  // every device entry point comes through here before touching the stream
    if (l < 1) return set_error(PM_ERR_INVALID_PARAMS, "motif length l must be positive");
    if (l > PM_MAX_L) {
        return set_error(PM_ERR_UNSUPPORTED, "l=" + std::to_string(l) + " exceeds this build's limit of " +
                                                 std::to_string(PM_MAX_L) + " (one 64-bit word per l-mer)");
    }
    if (c->win_l == l) return PM_OK;
    c->win_off.assign(static_cast<size_t>(c->t) + 1, 0);
    bool uniform = true;
    for (int i = 0; i < c->t; ++i) {
        const int64_t w = c->seq_len[static_cast<size_t>(i)] - l + 1;
        if (w < 1) {
            return set_error(PM_ERR_INVALID_PARAMS, "sequence 'seq" + std::to_string(i + 1) + "' of length " +
                                                        std::to_string(c->seq_len[static_cast<size_t>(i)]) +
                                                        " has no l-mer of length " + std::to_string(l));
        }
        c->win_off[static_cast<size_t>(i) + 1] = c->win_off[static_cast<size_t>(i)] + w;
        uniform = uniform && c->seq_len[static_cast<size_t>(i)] == c->seq_len[0];
    }
    c->x = c->win_off[static_cast<size_t>(c->t)];
    if (c->x > static_cast<int64_t>(std::numeric_limits<uint32_t>::max())) {
        return set_error(PM_ERR_INVALID_PARAMS, "sort-and-group hashing supports at most 2^32-1 l-mers");  // projection.hpp:284-287
    }
    c->uniform_w = uniform ? c->seq_len[0] - l + 1 : 0;
    // staging owned by the context (alive until the next change, which synchronises first): no sync here
    std::vector<double>& logw = c->h_logw;
    logw.resize(static_cast<size_t>(c->t));
    for (int i = 0; i < c->t; ++i) logw[static_cast<size_t>(i)] = std::log(static_cast<double>(c->seq_len[static_cast<size_t>(i)] - l + 1));
    PM_TRY(h2d(c, c->d_seq_logw, logw.data(), sizeof(double) * logw.size()));
    PM_TRY(h2d(c, c->d_win_off, c->win_off.data(), sizeof(int64_t) * (static_cast<size_t>(c->t) + 1)));
    c->win_l = l;
    return PM_OK;
}

// kept positions (1-based, validated) -> constant-memory extraction program
k::PlanProg make_prog(const int32_t* kept, int kk) {
    k::PlanProg pp;
    std::memset(&pp, 0, sizeof(pp));
    pp.keybits = static_cast<uint8_t>(2 * kk);
    int i = 0;
    while (i < kk) {
        int j = i;
        while (j + 1 < kk && kept[j + 1] == kept[j] + 1) ++j;
        const int width = j - i + 1;
        pp.rshift[pp.nruns] = static_cast<uint8_t>(64 - 2 * kept[j]);  // last digit of the run, 0-based kept[j]-1
        pp.nbits[pp.nruns] = static_cast<uint8_t>(2 * width);
        ++pp.nruns;
        i = j + 1;
    }
    return pp;
}

// ---------------------------------------------------------------------------------------------
// stable segmented radix sort driver: sorts key bits [0, keybits) of every segment; on return
// *ko/*io point at the buffers holding the result.
// ---------------------------------------------------------------------------------------------
template <typename KeyT>
int sort_segments(pm_ctx* c, KeyT* ka, KeyT* kb, unsigned int* ia, unsigned int* ib, int nseg, int64_t stride,
                  int64_t len, const unsigned int* len_dev, int keybits, KeyT** ko, unsigned int** io) {
    const int64_t span = len_dev ? stride : len;
    const int tiles = static_cast<int>((span + k::kSortTile - 1) / k::kSortTile);
    unsigned int* counts = nullptr;
    PM_TRY(get_buf(c, S_COUNTS, static_cast<size_t>(nseg) * 256 * static_cast<size_t>(std::max(tiles, 1)), &counts));
    const int passes = (keybits + 7) / 8;
    KeyT* kin = ka;
    KeyT* kout = kb;
    unsigned int* iin = ia;
    unsigned int* iout = ib;
    bool first = true;
    if (tiles == 0 || nseg == 0) {
        *ko = ka;
        *io = ia;
        return PM_OK;
    }
    for (int pass = 0; pass < passes; ++pass) {
        const int shift = 8 * pass;
        const dim3 grid(static_cast<unsigned>(tiles), static_cast<unsigned>(nseg));
        k::radix_hist_kernel<KeyT><<<grid, k::kSortWarps * 32, 0, c->stream>>>(kin, stride, len, len_dev, tiles, shift, counts);
        PM_TRY(check_launch(c, "radix_hist"));
        const unsigned int* digit_base = nullptr;
        if (tiles <= 64) {
            k::radix_scan_kernel<<<nseg, 256, 0, c->stream>>>(counts, tiles);
            PM_TRY(check_launch(c, "radix_scan"));
        } else {  // large segments: scan the 256 digit rows of a segment in parallel
            unsigned int* totals = nullptr;
            PM_TRY(get_buf(c, S_DIGIT_TOT, static_cast<size_t>(nseg) * 256, &totals));
            k::radix_scan_rows_kernel<<<dim3(256, static_cast<unsigned>(nseg)), 256, 0, c->stream>>>(counts, tiles, totals);
            PM_TRY(check_launch(c, "radix_scan_rows"));
            k::radix_digit_base_kernel<<<nseg, 256, 0, c->stream>>>(totals);
            PM_TRY(check_launch(c, "radix_digit_base"));
            digit_base = totals;
        }
        if (first) {
            k::radix_scatter_kernel<KeyT, true><<<grid, k::kSortWarps * 32, 0, c->stream>>>(
                kin, iin, kout, iout, stride, len, len_dev, tiles, shift, counts, digit_base);
        } else {
            k::radix_scatter_kernel<KeyT, false><<<grid, k::kSortWarps * 32, 0, c->stream>>>(
                kin, iin, kout, iout, stride, len, len_dev, tiles, shift, counts, digit_base);
        }
        PM_TRY(check_launch(c, "radix_scatter"));
        first = false;
        std::swap(kin, kout);
        std::swap(iin, iout);
    }
    *ko = kin;
    *io = iin;
    return PM_OK;
}

// The projection plans of a launch live in __constant__ memory (k::c_plans), which is ONE array per device, while
// every context uploads and launches on its own stream.  Uses are therefore chained per device: a context's upload
// waits (on the device, not the host) for the kernel of the previous user, whichever stream that ran on.
struct ConstPlans {
    std::mutex mu;
    cudaEvent_t last_use = nullptr;
};
ConstPlans& const_plans_of(int device) {
    static std::mutex mu;
    static std::map<int, ConstPlans*> slots;
    std::lock_guard<std::mutex> lock(mu);
    ConstPlans*& s = slots[device];
    if (s == nullptr) s = new ConstPlans();
    return *s;
}
class ConstPlansUse {
public:
    ConstPlansUse(int device, cudaStream_t stream) : slot_(const_plans_of(device)), lock_(slot_.mu), stream_(stream) {
        if (slot_.last_use == nullptr) {
            cudaEventCreateWithFlags(&slot_.last_use, cudaEventDisableTiming);
        } else {
            cudaStreamWaitEvent(stream_, slot_.last_use, 0);
        }
    }
    ~ConstPlansUse() { cudaEventRecord(slot_.last_use, stream_); }  // after the kernel that reads the plans

private:
    ConstPlans& slot_;
    std::lock_guard<std::mutex> lock_;
    cudaStream_t stream_;
};

// keys of n_trials plans -> sorted (key, flat index) per trial
template <typename KeyT>
struct Sorted {
    KeyT* keys = nullptr;
    unsigned int* idx = nullptr;
};

template <typename KeyT>
int project_keys(pm_ctx* c, const std::vector<k::PlanProg>& progs, KeyT* keys) {
    const int n = static_cast<int>(progs.size());
    for (int base = 0; base < n; base += k::kMaxConstPlans) {
        const int cnt = std::min(k::kMaxConstPlans, n - base);
        c->h2d_bytes += static_cast<int64_t>(sizeof(k::PlanProg)) * cnt;
        ConstPlansUse plans_use(c->device, c->stream);
        PM_CUDA(cudaMemcpyToSymbolAsync(k::c_plans, progs.data() + base, sizeof(k::PlanProg) * static_cast<size_t>(cnt),
                                        0, cudaMemcpyHostToDevice, c->stream));
        const unsigned gx = static_cast<unsigned>(std::min<int64_t>((c->x + 255) / 256, 4096));
        const dim3 grid(std::max(gx, 1u), static_cast<unsigned>(cnt));
        k::project_keys_kernel<KeyT><<<grid, 256, 0, c->stream>>>(c->d_words, c->d_word_off, c->d_win_off, c->t, c->x,
                                                                c->uniform_w, base, cnt, keys);
        PM_TRY(check_launch(c, "project_keys"));
    }
    return PM_OK;
}

template <typename KeyT>
int hash_and_sort(pm_ctx* c, const std::vector<k::PlanProg>& progs, int keybits, Sorted<KeyT>* out) {
    const size_t n = progs.size() * static_cast<size_t>(c->x);
    KeyT *ka, *kb;
    unsigned int *ia, *ib;
    PM_TRY(get_buf(c, S_KEYS_A, n, &ka));
    PM_TRY(get_buf(c, S_KEYS_B, n, &kb));
    PM_TRY(get_buf(c, S_IDX_A, n, &ia));
    PM_TRY(get_buf(c, S_IDX_B, n, &ib));
    PM_TRY(project_keys<KeyT>(c, progs, ka));
    return sort_segments<KeyT>(c, ka, kb, ia, ib, static_cast<int>(progs.size()), c->x, c->x, nullptr, keybits,
                               &out->keys, &out->idx);
}

struct Records {
    uint64_t* key = nullptr;
    unsigned int* start = nullptr;
    unsigned int* size = nullptr;
    unsigned int* n_rec = nullptr;
    int64_t cap_e = 0;
};

template <typename KeyT>
int find_enriched(pm_ctx* c, const Sorted<KeyT>& s, int n_trials, int thr, Records* r) {
    r->cap_e = std::max<int64_t>(1, c->x / thr);
    const size_t n = static_cast<size_t>(n_trials) * static_cast<size_t>(r->cap_e);
    PM_TRY(get_buf(c, S_REC_KEY, n, &r->key));
    PM_TRY(get_buf(c, S_REC_START, n, &r->start));
    PM_TRY(get_buf(c, S_REC_SIZE, n, &r->size));
    PM_TRY(get_buf(c, S_NREC, static_cast<size_t>(n_trials) + 1, &r->n_rec));
    const int etiles = static_cast<int>((c->x + k::kEnrichTile - 1) / k::kEnrichTile);
    unsigned int* tile_cnt = nullptr;
    PM_TRY(get_buf(c, S_ETILES, static_cast<size_t>(n_trials) * static_cast<size_t>(etiles), &tile_cnt));
    const dim3 grid(static_cast<unsigned>(etiles), static_cast<unsigned>(n_trials));
    k::enrich_kernel<KeyT, false><<<grid, 1024, 0, c->stream>>>(s.keys, c->x, thr, r->cap_e, etiles, tile_cnt, r->key, r->start, r->size);
    PM_TRY(check_launch(c, "enrich_count"));
    k::enrich_scan_kernel<<<n_trials, 1024, 0, c->stream>>>(tile_cnt, etiles, r->n_rec);
    PM_TRY(check_launch(c, "enrich_scan"));
    k::enrich_kernel<KeyT, true><<<grid, 1024, 0, c->stream>>>(s.keys, c->x, thr, r->cap_e, etiles, tile_cnt, r->key, r->start, r->size);
    return check_launch(c, "enrich_write");
}

// ---------------------------------------------------------------------------------------------
// EM launcher
// ---------------------------------------------------------------------------------------------
using EmKernel = void (*)(const k::EmParams);

template <int G>
EmKernel em_for() { return k::em_refine_kernel<G>; }

EmKernel em_kernel_for(int l) {
    switch ((l + 1) / 2) {
        case 1: return em_for<1>();
        case 2: return em_for<2>();
        case 3: return em_for<3>();
        case 4: return em_for<4>();
        case 5: return em_for<5>();
        case 6: return em_for<6>();
        case 7: return em_for<7>();
        case 8: return em_for<8>();
        case 9: return em_for<9>();
        case 10: return em_for<10>();
        case 11: return em_for<11>();
        case 12: return em_for<12>();
        case 13: return em_for<13>();
        case 14: return em_for<14>();
        case 15: return em_for<15>();
        default: return em_for<16>();
    }
}

using EmSmemKernel = void (*)(const k::EmParams, const k::EmSmemExtra);

template <int G>
EmSmemKernel em_pair_for() { return k::em_refine_pair_kernel<G>; }

EmSmemKernel em_pair_kernel_for(int l) {
    switch ((l + 1) / 2) {
        case 1: return em_pair_for<1>();
        case 2: return em_pair_for<2>();
        case 3: return em_pair_for<3>();
        case 4: return em_pair_for<4>();
        case 5: return em_pair_for<5>();
        case 6: return em_pair_for<6>();
        case 7: return em_pair_for<7>();
        case 8: return em_pair_for<8>();
        case 9: return em_pair_for<9>();
        case 10: return em_pair_for<10>();
        case 11: return em_pair_for<11>();
        case 12: return em_pair_for<12>();
        case 13: return em_pair_for<13>();
        case 14: return em_pair_for<14>();
        case 15: return em_pair_for<15>();
        default: return em_pair_for<16>();
    }
}

// must mirror the carve-up at the top of em_refine_pair_kernel
size_t em_pair_smem_bytes(int nwarps, int G, int l, int zcap, int t, int total_words, bool big) {
    // big: tpad = sequences per tile (metadata only), two word stages of total_words (= largest tile) each
    const size_t TH = 4 * (static_cast<size_t>(l) + 1);
    const size_t tpad = big ? static_cast<size_t>(k::kPairMaxSeqs) : ((static_cast<size_t>(t) + 1) & ~static_cast<size_t>(1));
    const size_t NV = 2 * G <= 16 ? 16 : 32;
    size_t b = 0;
    b += (2 * TH + 2 * TH + 2 * TH + 2 * static_cast<size_t>(nwarps) + 12) * 8;              // thd, D64, L64, llpart, dscal
    b += 16 * static_cast<size_t>(G) * 8;                                                    // T2
    b += (32 * static_cast<size_t>(G) + (16 + static_cast<size_t>(nwarps)) * NV + 2 * tpad + 4) * 4;  // Cq, cpart, mprev, ubs
    b += (256 + 8 + 20 + 16 + 4 * tpad) * 4;                                                 // prof, iscal, s_off, wrow, smeta
    b += 16;                                                                                 // cons_bits
    b += static_cast<size_t>(nwarps) * 2 * k::kPairNearCap * 2;                              // near_j
    b = (b + 15) & ~static_cast<size_t>(15);
    b += ((static_cast<size_t>(zcap) + 1) & ~static_cast<size_t>(1)) * 8;                    // zbuf (float2), 16-byte multiple
    b += static_cast<size_t>(total_words) * 8 * (big ? 2 : 1);                               // TMA word stage(s)
    b += 16;                                                                                 // mbarriers
    return b + 16;
}

int em_smem_warps_for(int t);

// Warps per CTA of the pair kernel: as for the one-bucket kernel, a divisor of t so that the E-step (warp per
// sequence) is balanced; 12 warps were measured equal (C1) or slower (C2: ten sequences per tile) than 10.
int em_pair_warps_for(int t) {
    if (const char* env = std::getenv("PM_B200_EM_WARPS")) {  // tuning knob
        const long v = std::atol(env);
        if (v >= 2 && v <= k::kPairMaxWarps) return static_cast<int>(v);
    }
    return em_smem_warps_for(t);
}

int em_smem_warps_for(int t) {
    if (const char* env = std::getenv("PM_B200_EM_WARPS")) {  // tuning knob
        const long v = std::atol(env);
        if (v >= 1 && v <= k::kEmSmemMaxWarps) return static_cast<int>(v);
    }
    for (int nw : {10, 8, 6, 5, 4}) {  // <= k::kEmSmemMaxWarps (the kernel's launch bound)
        if (t % nw == 0) return nw;
    }
    return t >= 16 ? 8 : 4;
}

size_t em_smem_bytes(int nwarps) {
    size_t b = 0;
    b += 128 * 4;                          // th
    b += 256 * 4;                          // T
    b += static_cast<size_t>(nwarps) * 128 * 4;  // part
    b += 128 * 4;                          // rawm
    b += static_cast<size_t>(nwarps) * 8;  // llpart
    b += 8 * 8;                            // dscal
    b += static_cast<size_t>(nwarps) * k::kCandCap * 8;  // cand_v
    b += static_cast<size_t>(nwarps) * k::kCandCap * 4;  // cand_w
    b += 128 * 4;                          // prof
    b += 4 * 4;                            // iscal
    b += 8;                                // cons_bits
    return b + 16;
}

int em_warps_for(int t) {
    if (t >= 64) return 8;
    if (t % 5 == 0 && t % 4 != 0) return 5;
    return 4;
}

// Function attributes are per process, not per context: the dynamic shared-memory limit of a kernel only ever
// grows (monotone, under a lock), so a launch configured by one context stays valid whatever another one set.
// cudaFuncSetAttribute applies to the CURRENT device: the raised limits are remembered per (device, kernel)
int ensure_dynamic_smem(const void* func, size_t bytes, bool max_carveout) {
    static std::mutex mu;
    static std::map<std::pair<int, const void*>, size_t> allowed;
    int device = 0;
    PM_CUDA(cudaGetDevice(&device));
    std::lock_guard<std::mutex> lock(mu);
    size_t& cur = allowed[std::make_pair(device, func)];
    if (bytes > cur) {
        PM_CUDA(cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes)));
        if (cur == 0 && max_carveout) {
            PM_CUDA(cudaFuncSetAttribute(func, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared));
        }
        cur = bytes;
    }
    return PM_OK;
}

struct EmOut {
    int32_t* score = nullptr;
    int32_t* iters = nullptr;
    double* expct = nullptr;
    uint64_t* cons = nullptr;
    int32_t* pos = nullptr;
    double* theta = nullptr;
    double* ll = nullptr;
};


// refine() in FP64 (pm_em_f64.cuh), one CTA per work item.  steps_only: exactly max_iters em_step()s from theta_in.
int launch_em_f64(pm_ctx* c, int l, int max_iters, double tol, const k::WorkDesc* work, unsigned int n_work,
                  const unsigned int* members, const EmOut& o, unsigned long long* d_scal, const double* theta_in,
                  bool steps_only, const unsigned int* out_map = nullptr, const unsigned int* n_work_dev = nullptr) {
    k::EmParams p;
    std::memset(&p, 0, sizeof(p));
    p.words = c->d_words;
    p.word_off = c->d_word_off;
    p.seq_len = c->d_seq_len;
    p.win_off = c->d_win_off;
    p.seq_sym = c->d_seq_sym;
    p.seq_logw = c->d_seq_logw;
    for (int r = 0; r < 4; ++r) p.tot_sym[r] = static_cast<double>(c->tot_sym[r]);
    p.tot_bases = static_cast<double>(c->total_bases);
    p.t = c->t;
    p.l = l;
    p.max_iters = max_iters;
    p.tol = tol;
    p.work = work;
    p.n_work_dev = n_work_dev;  // device-side count (re-runs of flagged buckets); n_work is then its upper bound
    p.n_work = n_work;
    p.members = members;
    p.out_score = o.score;
    p.out_iters = o.iters;
    p.out_exp = o.expct;
    p.out_cons = o.cons;
    p.out_pos = o.pos;
    p.out_theta = o.theta;
    p.out_ll = o.ll;
    p.iter_total = d_scal;
    p.error_flag = reinterpret_cast<unsigned int*>(d_scal + 1);
    p.out_map = out_map;
    p.theta_in = theta_in;
    k::F64Extra x;
    const size_t per_cta = static_cast<size_t>(std::max<int64_t>(c->x, 1));
    const unsigned int grid = static_cast<unsigned int>(std::max<size_t>(
        1, std::min<size_t>({static_cast<size_t>(n_work), static_cast<size_t>(n_work_dev ? c->sm_count / 2 : 2 * c->sm_count),
                             (512u << 20) / (per_cta * 8)})));
    PM_TRY(get_buf(c, S_F64_Z, per_cta * grid, &x.zbuf));
    x.x = c->x;
    x.steps_only = steps_only ? 1 : 0;
    k::em_refine_f64_kernel<<<grid, k::kF64Threads, 0, c->stream>>>(p, x);
    return check_launch(c, "em_refine_f64");
}

// ---- tensor-core EM kernel (pm_em_tc.cuh) ------------------------------------------------------------------
// PM_B200_EM_TC (test/tuning knob): 0 keeps every bucket on the pair kernel, 2 uses the tensor-core kernel even for
// a handful of buckets.  Default: the tensor-core kernel from kTcMinWork buckets on -- a 128-bucket tile takes about a
// millisecond of sequential passes however few tiles there are, while the pair kernel refines ~4,000 buckets per
// millisecond, so smaller batches are faster there.  The count is only known on the device: the kernel itself hands
// a small batch over (TcExtra.min_work).
constexpr unsigned int kTcMinWork = 4096;
int em_tc_mode() {
    const char* env = std::getenv("PM_B200_EM_TC");
    return env ? std::atoi(env) : 1;
}
bool em_tc_enabled(unsigned int n_work_bound) {
    const int v = em_tc_mode();
    return v >= 2 || (v == 1 && n_work_bound >= kTcMinWork);
}

int tc_kc_for(int l) { return std::max(8, 4 * ((l + 3) / 4)); }

// gathers the flagged work items of the tensor-core launch for the exact kernel
__global__ void tc_compact_kernel(const unsigned char* __restrict__ flag, const k::WorkDesc* __restrict__ work,
                                  const unsigned int* __restrict__ n_work_dev, unsigned int n_work_host,
                                  k::WorkDesc* __restrict__ out_work, unsigned int* __restrict__ out_map,
                                  unsigned int* __restrict__ counter) {
    const unsigned int n = n_work_dev ? *n_work_dev : n_work_host;
    const unsigned int lane = threadIdx.x & 31u;
    for (unsigned int base = (blockIdx.x * blockDim.x + threadIdx.x) & ~31u; base < n; base += gridDim.x * blockDim.x) {
        const unsigned int i = base + lane;
        const bool f = i < n && flag[i] != 0;
        const unsigned int ball = __ballot_sync(0xffffffffu, f);
        if (ball == 0) continue;
        unsigned int at = 0;
        if (lane == 0) at = atomicAdd(counter, static_cast<unsigned int>(__popc(ball)));
        at = __shfl_sync(0xffffffffu, at, 0);
        if (f) {
            const unsigned int o = at + __popc(ball & ((1u << lane) - 1u));
            out_work[o] = work[i];
            out_map[o] = i;
        }
    }
}

// One sweep of the tensor-core kernel as a list of blocks (see TcBlock): every sequence's even windows, then its
// odd windows, in runs of 16 columns, cut into blocks of at most NBLK columns.
int build_tc_blocks(pm_ctx* c, int l) {
    if (c->tc_l == l) return PM_OK;
    const int KC = tc_kc_for(l);
    const int NBLK = KC <= 16 ? 128 : 96;
    auto ru = [](int v, int m) { return (v + m - 1) / m * m; };
    c->h_tc_blocks.clear();
    for (int i = 0; i < c->t; ++i) {
        const int W = c->seq_len[static_cast<size_t>(i)] - l + 1;
        const int ne = (W + 1) / 2, no = W / 2;
        const int ce = ru(ne, 16), co = ru(no, 16);
        const int cp = ru(ce + co, 32);
        const int nb = (cp + NBLK - 1) / NBLK, units = cp / 32;
        int b0 = 0;
        for (int b = 0; b < nb; ++b) {
            const int ncols = 32 * (units / nb + (b < units % nb ? 1 : 0));
            k::TcBlock B;
            std::memset(&B, 0, sizeof(B));
            B.seq = static_cast<uint16_t>(i);
            B.ncols = static_cast<uint16_t>(ncols);
            B.first = b == 0;
            B.last = b == nb - 1;
            int ns = 0;
            const int e_lo = b0, e_hi = std::min(b0 + ncols, ce);
            if (e_lo < e_hi) {
                k::TcSeg& sg = B.seg[ns++];
                sg.par = 0;
                sg.i0 = static_cast<uint16_t>(e_lo);
                sg.n = static_cast<uint16_t>(e_hi - e_lo);
                sg.col = 0;
                sg.valid = static_cast<uint16_t>(std::max(0, std::min(ne - e_lo, e_hi - e_lo)));
            }
            const int o_lo = std::max(b0, ce), o_hi = std::min(b0 + ncols, ce + co);
            if (o_lo < o_hi) {
                k::TcSeg& sg = B.seg[ns++];
                sg.par = 1;
                sg.i0 = static_cast<uint16_t>(o_lo - ce);
                sg.n = static_cast<uint16_t>(o_hi - o_lo);
                sg.col = static_cast<uint16_t>(o_lo - b0);
                sg.valid = static_cast<uint16_t>(std::max(0, std::min(no - (o_lo - ce), o_hi - o_lo)));
            }
            c->h_tc_blocks.push_back(B);
            b0 += ncols;
        }
    }
    c->tc_n_blocks = static_cast<int>(c->h_tc_blocks.size());
    c->tc_g1_flops = 0;
    c->tc_g2_flops = 0;
    for (const k::TcBlock& B : c->h_tc_blocks) {
        for (const k::TcSeg& sg : B.seg) {
            c->tc_g1_flops += 2LL * k::kTcRows * sg.n * (4 * KC);
            c->tc_g2_flops += 2LL * 2 * k::kTcRows * ((sg.valid + 15) / 16 * 16) * (4 * KC);
        }
    }
    c->tc_e_positions = ru(c->max_seq_len + k::kTcEPad, 32);
    PM_TRY(get_buf(c, S_TC_BLOCKS, c->h_tc_blocks.size(), &c->d_tc_blocks));
    PM_TRY(h2d(c, c->d_tc_blocks, c->h_tc_blocks.data(), sizeof(k::TcBlock) * c->h_tc_blocks.size()));
    c->tc_l = l;
    return PM_OK;
}

using EmTcKernel = void (*)(const k::EmParams, const k::TcExtra);
EmTcKernel em_tc_kernel_for(int l) {
    switch (tc_kc_for(l)) {
        case 8: return k::em_refine_tc_kernel<8>;
        case 12: return k::em_refine_tc_kernel<12>;
        case 16: return k::em_refine_tc_kernel<16>;
        default: return k::em_refine_tc_kernel<20>;
    }
}

// scalars on the device: [0] iter_total (u64) [1] error flag (u32 in the low half) [2] buckets refined again by the FP64
// kernel (u32 in the low half) [3] buckets the tensor-core kernel
// handed to the exact kernel (u32 in the low half) [4..7] the same by reason (a bucket can have several)
int launch_em(pm_ctx* c, int l, int max_iters, double tol, double z_eps, const k::WorkDesc* work,
              const unsigned int* n_work_dev, unsigned int n_work_host, unsigned int n_work_bound,
              const unsigned int* members, const EmOut& o, unsigned long long* d_scal, int max_count = 1 << 30,
              const double* theta_in = nullptr) {
    k::EmParams p;
    std::memset(&p, 0, sizeof(p));
    p.words = c->d_words;
    p.word_off = c->d_word_off;
    p.seq_len = c->d_seq_len;
    p.win_off = c->d_win_off;
    p.seq_sym = c->d_seq_sym;
    p.seq_logw = c->d_seq_logw;
    for (int r = 0; r < 4; ++r) p.tot_sym[r] = static_cast<double>(c->tot_sym[r]);
    p.tot_bases = static_cast<double>(c->total_bases);
    p.t = c->t;
    p.l = l;
    p.max_iters = max_iters;
    p.tol = tol;
    const double eps = z_eps < 0.0 ? 9.313225746154785e-10 /* 2^-30 */ : z_eps;
    p.z_eps = static_cast<float>(eps);
    p.log_z_eps = eps > 0.0 ? static_cast<float>(std::log(eps)) : -INFINITY;
    p.work = work;
    p.n_work_dev = n_work_dev;
    p.n_work = n_work_host;
    p.members = members;
    p.out_score = o.score;
    p.out_iters = o.iters;
    p.out_exp = o.expct;
    p.out_cons = o.cons;
    p.out_pos = o.pos;
    p.out_theta = o.theta;
    p.out_ll = o.ll;
    p.iter_total = d_scal;
    p.error_flag = reinterpret_cast<unsigned int*>(d_scal + 1);
    p.phase_clk = d_scal + 8;
    p.out_map = nullptr;
    p.theta_in = theta_in;
    p.flag_exact = nullptr;
    c->tc_used = false;
    const k::WorkDesc* const work_all = work;  // the TC stage below narrows p.work to the buckets it flagged

    // the class-group index may still be under construction on the worker thread (finish_class_groups): the tensor-core
    // stage only needs to know that the set is a small one the pair kernel will accept, which the upload already knew
    bool pair_small;
    if (c->cls_pending && c->cls_hint_small) {
        pair_small = true;
    } else {
        PM_TRY(finish_class_groups(c));
        pair_small = c->zlen > 0 && c->max_seq_len < 65536 && c->max_tile_seqs <= k::kPairMaxSeqs &&
                     !(c->t > k::kPairMaxSeqs || c->total_words > k::kPairMaxWords);
    }
    // Tensor-core kernel (pm_em_tc.cuh): 128 buckets per CTA.  It decides every bucket whose discrete outputs are clear
    // of the FP32 error of its sums and flags the rest, which the pair kernel below then refines into the same slots.
    if (pair_small && em_tc_enabled(n_work_bound) && theta_in == nullptr && l <= k::kTcMaxL && c->t <= k::kTcMaxSeqs &&
        max_iters <= k::kTcMaxIters && max_count <= 255 && c->max_seq_len + k::kTcEPad <= 4096 && n_work_bound >= 1) {
        PM_TRY(build_tc_blocks(c, l));
        const size_t smem = std::max<size_t>(k::tc_smem_bytes(c->t, c->tc_n_blocks, c->tc_e_positions), 120 * 1024);
        if (smem <= 227 * 1024) {
            EmTcKernel kern = em_tc_kernel_for(l);
            PM_TRY(ensure_dynamic_smem(reinterpret_cast<const void*>(kern), smem, true));
            k::TcExtra x;
            x.blocks = c->d_tc_blocks;
            x.n_blocks = c->tc_n_blocks;
            x.e_positions = c->tc_e_positions;
            x.tie_delta = 1e-3f;
            x.ll_margin = 1e-2f;
            x.stats = d_scal + 4;
            x.min_work = em_tc_mode() >= 2 ? 0u : kTcMinWork;
            unsigned int* d_cnt = reinterpret_cast<unsigned int*>(d_scal + 3);  // zeroed by the caller with the other scalars
            k::WorkDesc* d_list;
            unsigned int* d_map;
            PM_TRY(get_buf(c, S_TC_FLAG, static_cast<size_t>(n_work_bound), &x.out_flag));
            PM_TRY(get_buf(c, S_TC_WORK, static_cast<size_t>(n_work_bound), &d_list));
            PM_TRY(get_buf(c, S_TC_MAP, static_cast<size_t>(n_work_bound), &d_map));
            const unsigned int tiles = (n_work_bound + k::kTcRows - 1) / k::kTcRows;
            const unsigned int grid = std::max(1u, std::min(static_cast<unsigned int>(c->sm_count), tiles));
            kern<<<grid, k::kTcThreads, smem, c->stream>>>(p, x);
            PM_TRY(check_launch(c, "em_refine_tc"));
            c->tc_used = true;
            const unsigned int cgrid = std::max(1u, std::min(1024u, (n_work_bound + 255) / 256));
            tc_compact_kernel<<<cgrid, 256, 0, c->stream>>>(x.out_flag, work, n_work_dev, n_work_host, d_list, d_map, d_cnt);
            PM_TRY(check_launch(c, "tc_compact"));
            // the exact kernel takes over the flagged buckets
            p.work = d_list;
            p.n_work_dev = d_cnt;
            p.n_work = 0;
            p.out_map = d_map;
        }
    }

    PM_TRY(finish_class_groups(c));
    const bool pair_ok = c->zlen > 0 && c->max_seq_len < 65536 && c->max_tile_seqs <= k::kPairMaxSeqs;
    if (pair_ok) {
        // two buckets per CTA in lockstep (pm_em_pair.cuh).  Small sets keep all per-sequence state and the whole
        // packed set in shared memory; large sets walk the tiles with per-tile state (C5: 1,000 tiles of 10).
        const bool big = c->t > k::kPairMaxSeqs || c->total_words > k::kPairMaxWords;
        const int G = (l + 1) / 2;
        const int nwarps = em_pair_warps_for(big ? std::min(c->max_tile_seqs, 10) : c->t);
        const int threads = nwarps * 32;
        const int stage_words = big ? c->tile_words : static_cast<int>(c->total_words);
        const size_t smem = em_pair_smem_bytes(nwarps, G, l, c->zlen, c->t, stage_words, big);
        if (smem <= 227 * 1024) {
            EmSmemKernel kern = em_pair_kernel_for(l);
            int per_sm = 0;
            if (c->pair_cfg_l == l && c->pair_cfg_smem == smem && c->pair_cfg_threads == threads) {
                per_sm = c->pair_cfg_per_sm;
            } else {
                PM_TRY(ensure_dynamic_smem(reinterpret_cast<const void*>(kern), smem, true));
                PM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem));
                c->pair_cfg_l = l;
                c->pair_cfg_smem = smem;
                c->pair_cfg_threads = threads;
                c->pair_cfg_per_sm = per_sm;
            }
            if (per_sm >= 1) {
                if (const char* env = std::getenv("PM_B200_EM_PER_SM")) {  // experiment knob: fewer resident CTAs
                    const long v = std::atol(env);
                    if (v >= 1 && v < per_sm) per_sm = static_cast<int>(v);
                }
                const unsigned int full = static_cast<unsigned int>(c->sm_count * per_sm);
                const unsigned int grid = std::max(1u, std::min(full, (n_work_bound + 1) / 2));
                k::EmSmemExtra x;
                x.tiles = c->d_tiles;
                x.n_tiles = c->n_tiles;
                x.cls_entries = c->d_cls_entries;
                x.tile_group_off = c->d_cls_group_off;
                x.seq_zoff = c->d_seq_zoff;
                x.mprev_g = nullptr;  // non-null selects the large-set path
                x.zcap = c->zlen;
                x.wcap = stage_words;
                if (big) PM_TRY(get_buf(c, S_MPREV, static_cast<size_t>(grid) * 2 * static_cast<size_t>(c->t), &x.mprev_g));
                // third tier: stop decisions within the error of this kernel's likelihood, and argmax decisions between
                // different windows whose FP64 weights agree to 1e-9, go to the FP64 kernel
                const bool tier3 = theta_in == nullptr;
                if (tier3) {
                    PM_TRY(get_buf(c, S_F64_FLAG, static_cast<size_t>(n_work_bound), &p.flag_exact));
                    PM_CUDA(cudaMemsetAsync(p.flag_exact, 0, static_cast<size_t>(n_work_bound), c->stream));
                }
                kern<<<grid, threads, smem, c->stream>>>(p, x);
                PM_TRY(check_launch(c, "em_refine_pair"));
                if (tier3) {
                    k::WorkDesc* d_list2;
                    unsigned int* d_map2;
                    unsigned int* d_cnt2 = reinterpret_cast<unsigned int*>(d_scal + 2);
                    PM_TRY(get_buf(c, S_F64_WORK, static_cast<size_t>(n_work_bound), &d_list2));
                    PM_TRY(get_buf(c, S_F64_MAP, static_cast<size_t>(n_work_bound), &d_map2));
                    const unsigned int cgrid = std::max(1u, std::min(1024u, (n_work_bound + 255) / 256));
                    tc_compact_kernel<<<cgrid, 256, 0, c->stream>>>(p.flag_exact, work_all, n_work_dev, n_work_host, d_list2, d_map2, d_cnt2);
                    PM_TRY(check_launch(c, "f64_compact"));
                    PM_TRY(launch_em_f64(c, l, max_iters, tol, d_list2, n_work_bound, members, o, d_scal, nullptr, false, d_map2, d_cnt2));
                }
                return PM_OK;
            }
        }
    }
    const int nwarps = em_warps_for(c->t);
    const int threads = nwarps * 32;
    const size_t smem = em_smem_bytes(nwarps);
    EmKernel kern = em_kernel_for(l);
    int per_sm = 0;
    PM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem));
    per_sm = std::max(per_sm, 1);
    const unsigned int full = static_cast<unsigned int>(c->sm_count * per_sm);
    const unsigned int grid = std::max(1u, std::min(full, n_work_bound));
    kern<<<grid, threads, smem, c->stream>>>(p);
    return check_launch(c, "em_refine");
}

void unpack_consensus(uint64_t bits, int l, char* out) {
    static const char sym[4] = {'A', 'C', 'T', 'G'};
    for (int c = 0; c < l; ++c) out[c] = sym[(bits >> (62 - 2 * c)) & 3];
    out[l] = '\0';
}

int pack_lmer(const char* v, int l, uint64_t* out) {
    uint64_t bits = 0;
    for (int c = 0; c < l; ++c) {
        int r;
        switch (v[c]) {
            case 'A': r = 0; break;
            case 'C': r = 1; break;
            case 'T': r = 2; break;
            case 'G': r = 3; break;
            default:
                return set_error(PM_ERR_UNKNOWN_SYMBOL, std::string("symbol '") + v[c] + "' is not in alphabet \"ACTG\"");
        }
        bits |= static_cast<uint64_t>(r) << (62 - 2 * c);
    }
    *out = bits;
    return PM_OK;
}

int check_backend(int backend, int kk, uint64_t dense_cap) {
    // projection.hpp:341-351: an explicit dense request above the cap is an error; results are
    // otherwise backend-independent, and this build always sorts.
    if (backend == PM_BACKEND_DENSE && pow4(kk) > dense_cap) {
        return set_error(PM_ERR_DENSE_TABLE_TOO_LARGE, "dense backend would allocate " + std::to_string(pow4(kk)) +
                                                           " buckets, above the cap of " + std::to_string(dense_cap) +
                                                           "; use the grouped backend");
    }
    return PM_OK;
}

int check_plan_for_hash(pm_ctx* c, int l, const int32_t* kept, int kk) {
    PM_TRY(need_sequences(c));
    PM_TRY(validate_plan(l, kept, kk));
    if (kk > 31) {
        return set_error(PM_ERR_KMER_TOO_LONG, "projection width " + std::to_string(kk) +
                                                   " exceeds the encodable k-mer length 31");  // projection.hpp:327-330
    }
    return prepare_windows(c, l);
}

}  // namespace

extern "C" {

int pm_ctx_create(int device, void* stream, pm_ctx** out) {
    clear_error();
    if (out == nullptr) return set_error(PM_ERR_INVALID_PARAMS, "null output pointer");
    int count = 0;
    const cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess || count < 1) {
        return set_error(PM_ERR_NO_DEVICE, std::string("no CUDA device available (") +
                                               (e != cudaSuccess ? cudaGetErrorString(e) : "device count 0") +
                                               "); libpm_b200 has no CPU fallback");
    }
    if (device < 0 || device >= count) return set_error(PM_ERR_NO_DEVICE, "CUDA device ordinal out of range");
    cudaDeviceProp prop;
    PM_CUDA(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10) {
        return set_error(PM_ERR_NO_DEVICE, std::string("device '") + prop.name + "' is sm_" + std::to_string(prop.major) +
                                               std::to_string(prop.minor) + "; this library is built for sm_100a only");
    }
    PM_CUDA(cudaSetDevice(device));
    pm_ctx* c = new pm_ctx();
    c->device = device;
    c->stream = static_cast<cudaStream_t>(stream);
    c->sm_count = prop.multiProcessorCount;
    *out = c;
    return PM_OK;
}

void pm_ctx_destroy(pm_ctx* c) {
    if (c == nullptr) return;
    if (c->cls_pending) {
        try {
            c->cls_job.get();
        } catch (const std::exception&) {
        }
    }
    cudaSetDevice(c->device);
    cudaStreamSynchronize(c->stream);
    for (DevBuf& b : c->buf) {
        if (b.p) cudaFree(b.p);
    }
    cudaFree(c->d_words);
    cudaFree(c->d_word_off);
    cudaFree(c->d_seq_len);
    cudaFree(c->d_seq_sym);
    cudaFree(c->d_tot_sym);
    cudaFree(c->d_win_off);
    cudaFree(c->d_seq_logw);
    if (c->h_pin) cudaFreeHost(c->h_pin);
    cudaFree(c->d_cls_entries);
    cudaFree(c->d_cls_group_off);
    cudaFree(c->d_seq_zoff);
    cudaFree(c->d_tiles);
    delete c;
}

}  // extern "C"

namespace {
// SequenceSet ctor + 2-bit encoding.  ascii_on_device: the bases already sit in the context's device ASCII buffer
// (pm_ctx_generate_planted wrote them there); `bases` is then the host copy the class-group index is built from.
int load_sequences(pm_ctx* c, const char* bases, const int64_t* offs, int t, bool ascii_on_device) {
    if (c == nullptr || bases == nullptr || offs == nullptr) return set_error(PM_ERR_INVALID_PARAMS, "null argument");
    if (t < 1) return set_error(PM_ERR_INVALID_PARAMS, "a sequence set needs at least one sequence");
    for (int i = 0; i < t; ++i) {
        if (offs[i + 1] <= offs[i]) return set_error(PM_ERR_INVALID_PARAMS, "sequence 'seq" + std::to_string(i + 1) + "' is empty");
        if (offs[i + 1] - offs[i] > INT32_MAX) return set_error(PM_ERR_UNSUPPORTED, "sequence longer than 2^31-1 bases");
    }
    PM_CUDA(cudaSetDevice(c->device));
    HostMarks up_marks;
    if (c->cls_pending) {  // the previous set's index build: its staging vectors are about to be reused
        c->cls_pending = false;
        try {
            c->cls_job.get();
        } catch (const std::exception&) {
        }
    }
    PM_CUDA(cudaStreamSynchronize(c->stream));
    up_marks.mark("upload: sync");
    c->t = 0;
    c->win_l = 0;
    c->tc_l = -1;
    c->zlen = 0;
    c->n_tiles = 0;
    c->total_groups = 0;
    // the cached EM launch setups stay valid: they are keyed by (l, shared-memory bytes, threads)

    const int64_t base0 = offs[0];
    std::vector<int64_t> rel(static_cast<size_t>(t) + 1), word_off(static_cast<size_t>(t) + 1, 0);
    std::vector<int32_t> len(static_cast<size_t>(t));
    int64_t max_words = 0;
    for (int i = 0; i <= t; ++i) rel[static_cast<size_t>(i)] = offs[i] - base0;
    for (int i = 0; i < t; ++i) {
        const int64_t n = rel[static_cast<size_t>(i) + 1] - rel[static_cast<size_t>(i)];
        len[static_cast<size_t>(i)] = static_cast<int32_t>(n);
        // +1 zero pad word (word a+1 of any window exists), rounded up to an even count so that every
        // sequence starts 16-byte aligned: tiles are staged into shared memory with TMA bulk copies
        const int64_t nw = ((n + 31) / 32 + 2) & ~static_cast<int64_t>(1);
        word_off[static_cast<size_t>(i) + 1] = word_off[static_cast<size_t>(i)] + nw;
        max_words = std::max(max_words, nw);
    }
    const int64_t total_bases = rel[static_cast<size_t>(t)];
    const int64_t total_words = word_off[static_cast<size_t>(t)] + 2;

    char* d_ascii = nullptr;
    int64_t* d_offs = nullptr;
    PM_TRY(get_buf(c, S_ASCII, static_cast<size_t>(total_bases), &d_ascii));
    PM_TRY(get_buf(c, S_OFFS, static_cast<size_t>(t) + 1, &d_offs));
    PM_TRY(ensure(c, &c->d_words, &c->cap_words, sizeof(uint64_t) * static_cast<size_t>(total_words)));
    PM_TRY(ensure(c, &c->d_word_off, &c->cap_word_off, sizeof(int64_t) * (static_cast<size_t>(t) + 1)));
    PM_TRY(ensure(c, &c->d_seq_len, &c->cap_seq_len, sizeof(int32_t) * static_cast<size_t>(t)));
    PM_TRY(ensure(c, &c->d_seq_sym, &c->cap_seq_sym, sizeof(unsigned int) * 4 * static_cast<size_t>(t)));
    PM_TRY(ensure(c, &c->d_tot_sym, &c->cap_tot_sym, sizeof(unsigned long long) * 8));
    PM_TRY(ensure(c, &c->d_win_off, &c->cap_win_off, sizeof(int64_t) * (static_cast<size_t>(t) + 1)));
    PM_TRY(ensure(c, &c->d_seq_logw, &c->cap_seq_logw, sizeof(double) * static_cast<size_t>(t)));
    if (!ascii_on_device) PM_TRY(h2d(c, d_ascii, bases + base0, static_cast<size_t>(total_bases)));
    PM_TRY(h2d(c, d_offs, rel.data(), sizeof(int64_t) * rel.size()));
    PM_TRY(h2d(c, c->d_word_off, word_off.data(), sizeof(int64_t) * word_off.size()));
    PM_TRY(h2d(c, c->d_seq_len, len.data(), sizeof(int32_t) * len.size()));
    PM_CUDA(cudaMemsetAsync(c->d_words, 0, sizeof(uint64_t) * static_cast<size_t>(total_words), c->stream));
    PM_CUDA(cudaMemsetAsync(c->d_seq_sym, 0, sizeof(unsigned int) * 4 * static_cast<size_t>(t), c->stream));
    PM_CUDA(cudaMemsetAsync(c->d_tot_sym, 0, sizeof(unsigned long long) * 4, c->stream));
    PM_CUDA(cudaMemsetAsync(c->d_tot_sym + 4, 0xFF, sizeof(unsigned long long), c->stream));

    const int warps_per_block = 8;
    const dim3 grid(static_cast<unsigned>(std::min<int64_t>((max_words + warps_per_block - 1) / warps_per_block, 65535)),
                    static_cast<unsigned>(std::min(t, 65535)));
    k::encode_kernel<<<grid, warps_per_block * 32, 0, c->stream>>>(d_ascii, d_offs, c->d_word_off, t, c->d_words,
                                                                 c->d_seq_sym, c->d_tot_sym, c->d_tot_sym + 4);
    PM_TRY(check_launch(c, "encode"));
    up_marks.mark("h2d+encode issued");
    // The class-group index (host arithmetic over every base, ~0.1 ms for 12,000 bases) is only needed by the pair kernel.
    // Small sets build it on a worker thread -- from a copy of the input, the caller's buffer is free after this call --
    // while this thread goes on to sample plans and launch the hashing and tensor-core kernels; launch_em() joins it.
    {
        const int64_t cap = class_tile_cap(total_bases, t);
        int64_t longest = 0;
        for (int i = 0; i < t; ++i) longest = std::max<int64_t>(longest, len[static_cast<size_t>(i)]);
        c->cls_hint_small = t <= k::kPairMaxSeqs && total_words <= k::kPairMaxWords && longest < 65536 &&
                            k::kZPad + 31 + longest <= cap;
        if (c->cls_hint_small && total_bases <= (1 << 20) && std::getenv("PM_B200_SYNC_CLASS_GROUPS") == nullptr) {
            c->cls_bases.assign(bases + base0, static_cast<size_t>(total_bases));
            c->cls_rel = rel;
            c->cls_word_off = word_off;
            c->cls_job = std::async(std::launch::async, [c, t]() { return class_groups_cpu(c, c->cls_bases.data(), c->cls_rel, c->cls_word_off, t); });
            c->cls_pending = true;
        } else {
            PM_TRY(class_groups_upload(c, class_groups_cpu(c, bases + base0, rel, word_off, t), t));
        }
    }
    up_marks.mark("class groups");
    unsigned long long host_tot[5];
    PM_TRY(d2h(c, host_tot, c->d_tot_sym, sizeof(host_tot)));
    PM_CUDA(cudaStreamSynchronize(c->stream));
    up_marks.mark("final sync");
    if (host_tot[4] != ULLONG_MAX) {
        const int64_t bad = static_cast<int64_t>(host_tot[4]);
        int seq = 0;
        while (seq + 1 < t && rel[static_cast<size_t>(seq) + 1] <= bad) ++seq;
        return set_error(PM_ERR_UNKNOWN_SYMBOL, std::string("symbol '") + bases[base0 + bad] + "' in sequence 'seq" +
                                                    std::to_string(seq + 1) + "' is not in alphabet \"ACTG\"");
    }
    for (int r = 0; r < 4; ++r) c->tot_sym[r] = host_tot[r];
    c->t = t;
    c->offs = rel;
    c->word_off = word_off;
    c->seq_len = len;
    c->total_bases = total_bases;
    c->total_words = total_words;
    c->max_seq_len = *std::max_element(len.begin(), len.end());
    return PM_OK;
}
}  // namespace

extern "C" {

int pm_ctx_set_sequences(pm_ctx* c, const char* bases, const int64_t* offs, int t) {
    clear_error();
    return load_sequences(c, bases, offs, t, false);
}

int pm_ctx_generate_planted(pm_ctx* c, int t, int n, int l, int d, uint64_t seed, char* bases_out, char* motif,
                            int32_t* positions) {
    clear_error();
    if (c == nullptr) return set_error(PM_ERR_INVALID_PARAMS, "null context");
    if (t < 1) return set_error(PM_ERR_INVALID_PARAMS, "need at least one sequence, got t=" + std::to_string(t));
    if (l < 1 || l > n) {
        return set_error(PM_ERR_INVALID_PARAMS, "need 1 <= l <= n, got l=" + std::to_string(l) + ", n=" + std::to_string(n));
    }
    if (d < 0 || d >= l) {
        return set_error(PM_ERR_INVALID_PARAMS, "need 0 <= d < l, got d=" + std::to_string(d) + ", l=" + std::to_string(l));
    }
    if (l > PM_MAX_L) return set_error(PM_ERR_UNSUPPORTED, "l exceeds this build's limit of 31");
    PM_CUDA(cudaSetDevice(c->device));
    PM_CUDA(cudaStreamSynchronize(c->stream));
    const int64_t per_seq = static_cast<int64_t>(n) + (n - l + 1 > 1 ? 1 : 0) + 2 * d;
    const int64_t n_draws = l + static_cast<int64_t>(t) * per_seq;
    const int64_t total_bases = static_cast<int64_t>(t) * n;
    uint64_t* d_draws;
    char* d_ascii;
    unsigned char* d_out;  // [0..3] rejected flag, [8..40) motif, [64..) positions
    PM_TRY(get_buf(c, S_DRAWS, static_cast<size_t>(n_draws), &d_draws));
    PM_TRY(get_buf(c, S_ASCII, static_cast<size_t>(total_bases), &d_ascii));
    PM_TRY(get_buf(c, S_PLANT_OUT, 64 + sizeof(int32_t) * static_cast<size_t>(t), &d_out));
    PM_CUDA(cudaMemsetAsync(d_out, 0, 64, c->stream));
    k::mt64_stream_kernel<<<1, k::kMtThreads, 0, c->stream>>>(seed, n_draws, d_draws);
    PM_TRY(check_launch(c, "mt64_stream"));
    k::planted_build_kernel<<<static_cast<unsigned>(std::min(t, 4 * c->sm_count)), 256, 0, c->stream>>>(
        d_draws, t, n, l, d, d_ascii, reinterpret_cast<char*>(d_out + 8), reinterpret_cast<int32_t*>(d_out + 64),
        reinterpret_cast<unsigned int*>(d_out));
    PM_TRY(check_launch(c, "planted_build"));
    // the host keeps a copy of the bases: the class-group index of the EM kernels is built there, and callers get the
    // instance back like from pm_generate_planted
    std::vector<unsigned char> head(64 + sizeof(int32_t) * static_cast<size_t>(t));
    std::vector<char> host_bases(static_cast<size_t>(total_bases));
    PM_TRY(d2h(c, head.data(), d_out, head.size()));
    PM_TRY(d2h(c, host_bases.data(), d_ascii, host_bases.size()));
    PM_CUDA(cudaStreamSynchronize(c->stream));
    unsigned int rejected = 0;
    std::memcpy(&rejected, head.data(), sizeof(rejected));
    if (rejected != 0) {
        return set_error(PM_ERR_UNSUPPORTED, "seed " + std::to_string(seed) + " makes the reference redraw a bounded value "
                         "(probability < 1e-16 per draw): generate this instance with pm_generate_planted");
    }
    if (motif) std::memcpy(motif, head.data() + 8, static_cast<size_t>(l));
    if (positions) std::memcpy(positions, head.data() + 64, sizeof(int32_t) * static_cast<size_t>(t));
    if (bases_out) std::memcpy(bases_out, host_bases.data(), host_bases.size());
    std::vector<int64_t> offs(static_cast<size_t>(t) + 1);
    for (int i = 0; i <= t; ++i) offs[static_cast<size_t>(i)] = static_cast<int64_t>(i) * n;
    return load_sequences(c, host_bases.data(), offs.data(), t, true);
}

int pm_ctx_num_sequences(const pm_ctx* c) { return c ? c->t : 0; }

int64_t pm_ctx_total_lmers(const pm_ctx* c, int l) {
    if (c == nullptr || c->t < 1) return -1;
    int64_t x = 0;
    for (int i = 0; i < c->t; ++i) {
        const int64_t w = c->seq_len[static_cast<size_t>(i)] - l + 1;
        if (l < 1 || w < 1) return -1;
        x += w;
    }
    return x;
}

int pm_ctx_packed_words(pm_ctx* c, uint64_t* words_out, int64_t* word_off_out, int64_t cap_words) {
    clear_error();
    PM_TRY(need_sequences(c));
    const int64_t n = c->word_off[static_cast<size_t>(c->t)];
    if (cap_words < n) return set_error(PM_ERR_INVALID_PARAMS, "output buffer too small for the packed words");
    PM_CUDA(cudaSetDevice(c->device));
    PM_TRY(d2h(c, words_out, c->d_words, sizeof(uint64_t) * static_cast<size_t>(n)));
    PM_CUDA(cudaStreamSynchronize(c->stream));
    std::memcpy(word_off_out, c->word_off.data(), sizeof(int64_t) * c->word_off.size());
    return PM_OK;
}

int pm_ctx_symbol_counts(pm_ctx* c, int64_t* counts4) {
    clear_error();
    PM_TRY(need_sequences(c));
    for (int r = 0; r < 4; ++r) counts4[r] = static_cast<int64_t>(c->tot_sym[r]);
    return PM_OK;
}

int pm_ctx_synchronize(pm_ctx* c) {
    clear_error();
    if (c == nullptr) return set_error(PM_ERR_INVALID_PARAMS, "null context");
    PM_CUDA(cudaSetDevice(c->device));
    PM_CUDA(cudaStreamSynchronize(c->stream));
    return PM_OK;
}

int pm_ctx_em_exact_counts(const pm_ctx* c, int64_t* out6) {
    if (c == nullptr || out6 == nullptr) return set_error(PM_ERR_INVALID_PARAMS, "null argument");
    for (int i = 0; i < 6; ++i) out6[i] = c->em_exact[i];
    return PM_OK;
}

int64_t pm_ctx_launch_count(const pm_ctx* c) { return c ? c->launches : 0; }

// ------------------------------------------------------------------------------------------------
// stage entry points
// ------------------------------------------------------------------------------------------------
int pm_hash_keys(pm_ctx* c, int l, const int32_t* kept, int kk, uint64_t* keys_out) {
    clear_error();
    PM_TRY(check_plan_for_hash(c, l, kept, kk));
    PM_CUDA(cudaSetDevice(c->device));
    const std::vector<k::PlanProg> progs(1, make_prog(kept, kk));
    uint64_t* keys = nullptr;
    PM_TRY(get_buf(c, S_KEYS_A, static_cast<size_t>(c->x), &keys));
    PM_TRY(project_keys<uint64_t>(c, progs, keys));
    PM_TRY(d2h(c, keys_out, keys, sizeof(uint64_t) * static_cast<size_t>(c->x)));
    PM_CUDA(cudaStreamSynchronize(c->stream));
    return PM_OK;
}

}  // extern "C"

namespace {

// hash_trial + bucket listing for one plan.  thr = 1 lists every bucket (hash_trial); order_by_size
// additionally applies the enriched_buckets ordering on the device.
template <typename KeyT>
int stage_buckets(pm_ctx* c, const int32_t* kept, int kk, int thr, bool order_by_size, std::vector<uint64_t>* keys,
                  std::vector<uint32_t>* starts, std::vector<uint32_t>* sizes, std::vector<uint32_t>* sorted_idx) {
    const std::vector<k::PlanProg> progs(1, make_prog(kept, kk));
    Sorted<KeyT> srt;
    PM_TRY(hash_and_sort<KeyT>(c, progs, 2 * kk, &srt));
    Records rec;
    PM_TRY(find_enriched<KeyT>(c, srt, 1, thr, &rec));
    unsigned int n_rec = 0;
    PM_TRY(d2h(c, &n_rec, rec.n_rec, sizeof(n_rec)));
    PM_CUDA(cudaStreamSynchronize(c->stream));
    const size_t ne = n_rec;
    std::vector<uint32_t> order(ne);
    for (size_t i = 0; i < ne; ++i) order[i] = static_cast<uint32_t>(i);
    if (order_by_size && ne > 1) {
        // stable sort of the records by (x - size): equal sizes keep their ascending-key order
        unsigned int *ka, *kb, *ia, *ib;
        PM_TRY(get_buf(c, S_TMP_A, static_cast<size_t>(rec.cap_e), &ka));
        PM_TRY(get_buf(c, S_TMP_B, static_cast<size_t>(rec.cap_e), &kb));
        PM_TRY(get_buf(c, S_TMP_C, static_cast<size_t>(rec.cap_e), &ia));
        PM_TRY(get_buf(c, S_TMP_D, static_cast<size_t>(rec.cap_e), &ib));
        const unsigned gx = static_cast<unsigned>(std::min<int64_t>((rec.cap_e + 255) / 256, 1024));
        k::size_keys_kernel<<<dim3(gx, 1), 256, 0, c->stream>>>(rec.size, rec.n_rec, rec.cap_e,
                                                              static_cast<unsigned int>(c->x), 1, ka);
        PM_TRY(check_launch(c, "size_keys"));
        int bits = 1;
        while ((static_cast<uint64_t>(c->x) >> bits) != 0) ++bits;
        unsigned int* ko;
        unsigned int* io;
        PM_TRY((sort_segments<unsigned int>(c, ka, kb, ia, ib, 1, rec.cap_e, rec.cap_e, rec.n_rec, bits, &ko, &io)));
        PM_TRY(d2h(c, order.data(), io, sizeof(uint32_t) * ne));
        PM_CUDA(cudaStreamSynchronize(c->stream));
    }
    std::vector<uint64_t> hk(ne);
    std::vector<uint32_t> hs(ne), hz(ne);
    sorted_idx->resize(static_cast<size_t>(c->x));
    PM_TRY(d2h(c, hk.data(), rec.key, sizeof(uint64_t) * ne));
    PM_TRY(d2h(c, hs.data(), rec.start, sizeof(uint32_t) * ne));
    PM_TRY(d2h(c, hz.data(), rec.size, sizeof(uint32_t) * ne));
    PM_TRY(d2h(c, sorted_idx->data(), srt.idx, sizeof(uint32_t) * static_cast<size_t>(c->x)));
    PM_CUDA(cudaStreamSynchronize(c->stream));
    keys->resize(ne);
    starts->resize(ne);
    sizes->resize(ne);
    for (size_t i = 0; i < ne; ++i) {
        (*keys)[i] = hk[order[i]];
        (*starts)[i] = hs[order[i]];
        (*sizes)[i] = hz[order[i]];
    }
    return PM_OK;
}

int stage_buckets_any(pm_ctx* c, const int32_t* kept, int kk, int thr, bool order_by_size, std::vector<uint64_t>* keys,
                      std::vector<uint32_t>* starts, std::vector<uint32_t>* sizes, std::vector<uint32_t>* sorted_idx) {
    if (2 * kk <= 32) return stage_buckets<uint32_t>(c, kept, kk, thr, order_by_size, keys, starts, sizes, sorted_idx);
    return stage_buckets<uint64_t>(c, kept, kk, thr, order_by_size, keys, starts, sizes, sorted_idx);
}

}  // namespace

extern "C" {

int pm_hash_trial(pm_ctx* c, int l, const int32_t* kept, int kk, int backend, uint64_t dense_table_cap,
                  int64_t* n_buckets, uint64_t* bucket_keys, int32_t* bucket_sizes, int32_t* members) {
    clear_error();
    PM_TRY(check_plan_for_hash(c, l, kept, kk));
    PM_TRY(check_backend(backend, kk, dense_table_cap));
    PM_CUDA(cudaSetDevice(c->device));
    std::vector<uint64_t> keys;
    std::vector<uint32_t> starts, sizes, idx;
    PM_TRY(stage_buckets_any(c, kept, kk, 1, false, &keys, &starts, &sizes, &idx));
    *n_buckets = static_cast<int64_t>(keys.size());
    for (size_t b = 0; b < keys.size(); ++b) {
        bucket_keys[b] = keys[b];
        bucket_sizes[b] = static_cast<int32_t>(sizes[b]);
    }
    for (size_t i = 0; i < idx.size(); ++i) members[i] = static_cast<int32_t>(idx[i]);
    return PM_OK;
}

int pm_enriched_buckets(pm_ctx* c, int l, const int32_t* kept, int kk, int s, int r_cap, int64_t* n_enriched,
                        uint64_t* keys_out, int32_t* sizes_pre, int32_t* overflowed, int64_t* mem_off, int32_t* members) {
    clear_error();
    PM_TRY(check_plan_for_hash(c, l, kept, kk));
    if (s < 1 || r_cap < s) return set_error(PM_ERR_INVALID_PARAMS, "enriched buckets need s >= 1 and r_cap >= s");
    PM_CUDA(cudaSetDevice(c->device));
    std::vector<uint64_t> keys;
    std::vector<uint32_t> starts, sizes, idx;
    PM_TRY(stage_buckets_any(c, kept, kk, s, true, &keys, &starts, &sizes, &idx));
    *n_enriched = static_cast<int64_t>(keys.size());
    int64_t pos = 0;
    for (size_t b = 0; b < keys.size(); ++b) {
        keys_out[b] = keys[b];
        sizes_pre[b] = static_cast<int32_t>(sizes[b]);
        overflowed[b] = sizes[b] > static_cast<uint32_t>(r_cap) ? 1 : 0;
        const uint32_t take = std::min(sizes[b], static_cast<uint32_t>(r_cap));
        mem_off[b] = pos;
        for (uint32_t m = 0; m < take; ++m) members[pos++] = static_cast<int32_t>(idx[starts[b] + m]);
    }
    mem_off[keys.size()] = pos;
    return PM_OK;
}

}  // extern "C"

namespace {

// refine() for n_buckets member lists: the production kernels (exact == false) or the FP64 kernel; theta_in
// (n_buckets models) replaces init_model and steps_only turns the call into max_iters em_step()s.
int refine_common(pm_ctx* c, int l, const int32_t* members, const int64_t* mem_off, int n_buckets, int max_iters,
                  double tol, double z_epsilon, bool exact, const double* theta_in, bool steps_only, char* consensus,
                  int32_t* positions, int32_t* score, double* expectation, int32_t* iterations, double* theta,
                  double* ll_trace) {
    clear_error();
    PM_TRY(need_sequences(c));
    if (c != nullptr) PM_CUDA(cudaSetDevice(c->device));
    PM_TRY(prepare_windows(c, l));
    if (max_iters < 1) return set_error(PM_ERR_INVALID_PARAMS, "need at least one EM iteration");
    if (n_buckets < 1) return PM_OK;
    const int64_t n_mem = mem_off ? mem_off[n_buckets] : 0;
    std::vector<k::WorkDesc> work(static_cast<size_t>(n_buckets));
    for (int b = 0; b < n_buckets; ++b) {
        const int64_t cnt = mem_off ? mem_off[b + 1] - mem_off[b] : 0;
        if (cnt < 1 && theta_in == nullptr) return set_error(PM_ERR_EMPTY_BUCKET, "cannot build a motif model from an empty bucket");
        work[static_cast<size_t>(b)].mem_begin = mem_off ? mem_off[b] : 0;
        work[static_cast<size_t>(b)].key = 0;
        work[static_cast<size_t>(b)].count = static_cast<unsigned int>(cnt);
        work[static_cast<size_t>(b)].trial = b;
    }
    for (int64_t i = 0; i < n_mem; ++i) {
        if (members[i] < 0 || members[i] >= c->x) return set_error(PM_ERR_INDEX_OUT_OF_RANGE, "member l-mer index out of range");
    }
    const size_t nb = static_cast<size_t>(n_buckets);
    const size_t TH = 4 * static_cast<size_t>(l + 1);
    unsigned int* d_mem;
    k::WorkDesc* d_work;
    unsigned long long* d_scal;
    double* d_theta_in = nullptr;
    EmOut o;
    const bool xs = exact;  // scratch set
    PM_TRY(get_buf(c, xs ? S_X_MEMBERS : S_MEMBERS, static_cast<size_t>(std::max<int64_t>(n_mem, 1)), &d_mem));
    PM_TRY(get_buf(c, xs ? S_X_WORK : S_WORK, nb, &d_work));
    PM_TRY(get_buf(c, xs ? S_X_SCAL : S_SCAL, 16, &d_scal));
    PM_TRY(get_buf(c, xs ? S_X_SCORE : S_OUT_SCORE, nb, &o.score));
    PM_TRY(get_buf(c, xs ? S_X_ITERS : S_OUT_ITERS, nb, &o.iters));
    PM_TRY(get_buf(c, xs ? S_X_EXP : S_OUT_EXP, nb, &o.expct));
    PM_TRY(get_buf(c, xs ? S_X_CONS : S_OUT_CONS, nb, &o.cons));
    PM_TRY(get_buf(c, xs ? S_X_POS : S_OUT_POS, nb * static_cast<size_t>(c->t), &o.pos));
    if (theta) PM_TRY(get_buf(c, xs ? S_X_THETA : S_OUT_THETA, nb * TH, &o.theta));
    if (theta_in) {
        PM_TRY(get_buf(c, xs ? S_X_THETA_IN : S_THETA_IN, nb * TH, &d_theta_in));
        PM_TRY(h2d(c, d_theta_in, theta_in, sizeof(double) * nb * TH));
    }
    if (ll_trace) {
        PM_TRY(get_buf(c, xs ? S_X_LL : S_OUT_LL, nb * static_cast<size_t>(max_iters), &o.ll));
        std::vector<double> nan_fill(nb * static_cast<size_t>(max_iters), std::numeric_limits<double>::quiet_NaN());
        PM_TRY(h2d(c, o.ll, nan_fill.data(), sizeof(double) * nan_fill.size()));
        PM_CUDA(cudaStreamSynchronize(c->stream));
    }
    if (n_mem > 0) PM_TRY(h2d(c, d_mem, members, sizeof(int32_t) * static_cast<size_t>(n_mem)));
    PM_TRY(h2d(c, d_work, work.data(), sizeof(k::WorkDesc) * nb));
    PM_CUDA(cudaMemsetAsync(d_scal, 0, sizeof(unsigned long long) * 16, c->stream));
    if (exact) {
        PM_TRY(launch_em_f64(c, l, max_iters, tol, d_work, static_cast<unsigned int>(n_buckets), d_mem, o, d_scal, d_theta_in,
                             steps_only));
    } else {
        unsigned int max_count = 0;
        for (const k::WorkDesc& w : work) max_count = std::max(max_count, w.count);
        PM_TRY(launch_em(c, l, max_iters, tol, z_epsilon, d_work, nullptr, static_cast<unsigned int>(n_buckets),
                         static_cast<unsigned int>(n_buckets), d_mem, o, d_scal,
                         static_cast<int>(std::min<unsigned int>(max_count, 1u << 30)), d_theta_in));
    }
    std::vector<int32_t> hs(nb), hi(nb);
    std::vector<double> he(nb);
    std::vector<uint64_t> hc(nb);
    unsigned long long scal[8];
    PM_TRY(d2h(c, hs.data(), o.score, sizeof(int32_t) * nb));
    PM_TRY(d2h(c, hi.data(), o.iters, sizeof(int32_t) * nb));
    PM_TRY(d2h(c, he.data(), o.expct, sizeof(double) * nb));
    PM_TRY(d2h(c, hc.data(), o.cons, sizeof(uint64_t) * nb));
    PM_TRY(d2h(c, scal, d_scal, sizeof(scal)));
    if (positions) PM_TRY(d2h(c, positions, o.pos, sizeof(int32_t) * nb * static_cast<size_t>(c->t)));
    if (theta) PM_TRY(d2h(c, theta, o.theta, sizeof(double) * nb * TH));
    if (ll_trace) PM_TRY(d2h(c, ll_trace, o.ll, sizeof(double) * nb * static_cast<size_t>(max_iters)));
    PM_CUDA(cudaStreamSynchronize(c->stream));
    if (!exact) {
        if ((scal[4] | scal[5] | scal[6] | scal[7]) == 0) scal[3] = 0;  // a small batch handed over wholesale
        c->em_exact[0] = static_cast<int64_t>(scal[3] & 0xFFFFFFFFULL);
        for (int r = 0; r < 4; ++r) c->em_exact[1 + r] = static_cast<int64_t>(scal[4 + r]);
        c->em_exact[5] = static_cast<int64_t>(scal[2] & 0xFFFFFFFFULL);
    }
    if ((scal[1] & 0xFFFFFFFFULL) != 0) {
        return set_error(PM_ERR_NUMERICAL_UNDERFLOW, "all window weights vanished in some sequence");
    }
    for (size_t b = 0; b < nb; ++b) {
        if (score) score[b] = hs[b];
        if (iterations) iterations[b] = hi[b];
        if (expectation) expectation[b] = he[b];
        if (consensus) unpack_consensus(hc[b], l, consensus + 32 * b);
    }
    return PM_OK;
}

}  // namespace

extern "C" {

int pm_refine(pm_ctx* c, int l, const int32_t* members, const int64_t* mem_off, int n_buckets, int max_iters,
              double tol, double z_epsilon, char* consensus, int32_t* positions, int32_t* score, double* expectation,
              int32_t* iterations, double* theta, double* ll_trace) {
    return refine_common(c, l, members, mem_off, n_buckets, max_iters, tol, z_epsilon, false, nullptr, false, consensus,
                         positions, score, expectation, iterations, theta, ll_trace);
}

int pm_refine_exact(pm_ctx* c, int l, const int32_t* members, const int64_t* mem_off, int n_buckets, int max_iters,
                    double tol, char* consensus, int32_t* positions, int32_t* score, double* expectation,
                    int32_t* iterations, double* theta, double* ll_trace) {
    return refine_common(c, l, members, mem_off, n_buckets, max_iters, tol, -1.0, true, nullptr, false, consensus, positions,
                         score, expectation, iterations, theta, ll_trace);
}

int pm_init_model(pm_ctx* c, int l, const int32_t* members, int n_members, double pseudocount, double* theta_out) {
    clear_error();
    PM_TRY(need_sequences(c));
    PM_CUDA(cudaSetDevice(c->device));
    PM_TRY(prepare_windows(c, l));
    if (theta_out == nullptr) return set_error(PM_ERR_INVALID_PARAMS, "null argument");
    if (n_members < 1) return set_error(PM_ERR_EMPTY_BUCKET, "cannot build a motif model from an empty bucket");
    if (!(pseudocount >= 0.0)) return set_error(PM_ERR_INVALID_PARAMS, "pseudocount must be non-negative");
    for (int i = 0; i < n_members; ++i) {
        if (members[i] < 0 || members[i] >= c->x) return set_error(PM_ERR_INDEX_OUT_OF_RANGE, "member l-mer index out of range");
    }
    const size_t TH = 4 * static_cast<size_t>(l + 1);
    k::WorkDesc wd{0, 0, static_cast<unsigned int>(n_members), 0};
    unsigned int* d_mem;
    k::WorkDesc* d_work;
    double* d_theta;
    PM_TRY(get_buf(c, S_MEMBERS, static_cast<size_t>(n_members), &d_mem));
    PM_TRY(get_buf(c, S_WORK, 1, &d_work));
    PM_TRY(get_buf(c, S_OUT_THETA, TH, &d_theta));
    PM_TRY(h2d(c, d_mem, members, sizeof(int32_t) * static_cast<size_t>(n_members)));
    PM_TRY(h2d(c, d_work, &wd, sizeof(wd)));
    k::EmParams p;
    std::memset(&p, 0, sizeof(p));
    p.words = c->d_words;
    p.word_off = c->d_word_off;
    p.win_off = c->d_win_off;
    for (int r = 0; r < 4; ++r) p.tot_sym[r] = static_cast<double>(c->tot_sym[r]);
    p.tot_bases = static_cast<double>(c->total_bases);
    p.t = c->t;
    p.l = l;
    p.work = d_work;
    p.n_work = 1;
    p.members = d_mem;
    p.out_theta = d_theta;
    k::init_model_kernel<<<1, 128, 0, c->stream>>>(p, pseudocount);
    PM_TRY(check_launch(c, "init_model"));
    PM_TRY(d2h(c, theta_out, d_theta, sizeof(double) * TH));
    PM_CUDA(cudaStreamSynchronize(c->stream));
    return PM_OK;
}

static int em_step_common(pm_ctx* c, int l, const double* theta_in, double* theta_out, double* log_likelihood, bool exact) {
    if (theta_in == nullptr || theta_out == nullptr) return set_error(PM_ERR_INVALID_PARAMS, "null argument");
    double ll = 0.0;
    // one em_step() = one iteration from theta_in: theta' and the likelihood of theta_in (refine.hpp:209, :281)
    const int rc = refine_common(c, l, nullptr, nullptr, 1, 1, 0.0, -1.0, exact, theta_in, exact, nullptr, nullptr, nullptr,
                                 nullptr, nullptr, theta_out, &ll);
    if (rc == PM_OK && log_likelihood) *log_likelihood = ll;
    return rc;
}

int pm_em_step(pm_ctx* c, int l, const double* theta_in, double* theta_out, double* log_likelihood) {
    return em_step_common(c, l, theta_in, theta_out, log_likelihood, false);
}

int pm_em_step_exact(pm_ctx* c, int l, const double* theta_in, double* theta_out, double* log_likelihood) {
    return em_step_common(c, l, theta_in, theta_out, log_likelihood, true);
}

int pm_expectation(const double* theta, int l, double* out) {
    clear_error();
    if (theta == nullptr || out == nullptr || l < 1) return set_error(PM_ERR_INVALID_PARAMS, "null argument");
    double sum = 0.0;
    for (int c = 1; c <= l; ++c) {  // refine.hpp:130-136: sum over motif columns of the column maximum
        double mx = theta[c];
        for (int r = 1; r < 4; ++r) mx = std::max(mx, theta[static_cast<size_t>(r) * (l + 1) + c]);
        sum += mx;
    }
    *out = sum;
    return PM_OK;
}

int pm_score(pm_ctx* c, int l, const int32_t* starts, int* score, char* consensus) {
    clear_error();
    PM_TRY(need_sequences(c));
    PM_TRY(prepare_windows(c, l));
    std::vector<int32_t> s0(static_cast<size_t>(c->t));
    for (int i = 0; i < c->t; ++i) {
        if (starts[i] < 1 || starts[i] + l - 1 > c->seq_len[static_cast<size_t>(i)]) {
            return set_error(PM_ERR_INDEX_OUT_OF_RANGE, "l-mer (i=" + std::to_string(i + 1) + ", j=" + std::to_string(starts[i]) +
                                                            ", l=" + std::to_string(l) + ") is out of range");
        }
        s0[static_cast<size_t>(i)] = starts[i] - 1;
    }
    PM_CUDA(cudaSetDevice(c->device));
    int32_t* d_starts;
    unsigned long long* d_out;
    PM_TRY(get_buf(c, S_TMP_A, static_cast<size_t>(c->t), &d_starts));
    PM_TRY(get_buf(c, S_SCAL, 4, &d_out));
    PM_TRY(h2d(c, d_starts, s0.data(), sizeof(int32_t) * s0.size()));
    k::score_kernel<<<1, 256, 0, c->stream>>>(c->d_words, c->d_word_off, c->t, l, d_starts,
                                            reinterpret_cast<int32_t*>(d_out), reinterpret_cast<uint64_t*>(d_out + 1));
    PM_TRY(check_launch(c, "score"));
    unsigned long long h[2];
    PM_TRY(d2h(c, h, d_out, sizeof(h)));
    PM_CUDA(cudaStreamSynchronize(c->stream));
    *score = static_cast<int>(h[0] & 0xFFFFFFFFULL);
    unpack_consensus(h[1], l, consensus);
    return PM_OK;
}

int pm_hamming_scan(pm_ctx* c, const char* v, int l, int d, int32_t* per_seq_min, int* total_distance, int* within_d) {
    clear_error();
    PM_TRY(need_sequences(c));
    PM_TRY(prepare_windows(c, l));
    uint64_t cand = 0;
    PM_TRY(pack_lmer(v, l, &cand));
    PM_CUDA(cudaSetDevice(c->device));
    int32_t* d_min;
    PM_TRY(get_buf(c, S_TMP_A, static_cast<size_t>(c->t), &d_min));
    const int threads = 256;
    const int blocks = std::max(1, std::min((c->t * 32 + threads - 1) / threads, c->sm_count * 8));
    k::hamming_scan_kernel<<<blocks, threads, 0, c->stream>>>(c->d_words, c->d_word_off, c->d_seq_len, c->t, l, cand, d_min);
    PM_TRY(check_launch(c, "hamming_scan"));
    std::vector<int32_t> h(static_cast<size_t>(c->t));
    PM_TRY(d2h(c, h.data(), d_min, sizeof(int32_t) * h.size()));
    PM_CUDA(cudaStreamSynchronize(c->stream));
    int tot = 0, within = 0;
    for (int i = 0; i < c->t; ++i) {
        tot += h[static_cast<size_t>(i)];
        within += h[static_cast<size_t>(i)] <= d ? 1 : 0;
        if (per_seq_min) per_seq_min[i] = h[static_cast<size_t>(i)];
    }
    if (total_distance) *total_distance = tot;
    if (within_d) *within_d = within;
    return PM_OK;
}

int pm_median_string(pm_ctx* c, int l, uint64_t limit, char* median, int* total_distance) {
    clear_error();
    PM_TRY(need_sequences(c));
    if (median == nullptr || total_distance == nullptr) return set_error(PM_ERR_INVALID_PARAMS, "null output pointer");
    if (l < 1 || l > 31) return set_error(PM_ERR_INVALID_PARAMS, "median string needs 1 <= l <= 31");  // oracle.hpp:122-124
    PM_TRY(prepare_windows(c, l));  // every n_i >= l (oracle.hpp:125-127)
    const uint64_t candidates = pow4(l);
    if (candidates > limit) {
        return set_error(PM_ERR_SEARCH_SPACE_TOO_LARGE, "median search needs " + std::to_string(candidates) +
                                                            " candidates, above the limit of " + std::to_string(limit));
    }
    if (l > 16) return set_error(PM_ERR_UNSUPPORTED, "median string on the device is limited to l <= 16 (32-bit candidate codes)");
    PM_CUDA(cudaSetDevice(c->device));
    unsigned long long* d_best;
    PM_TRY(get_buf(c, S_TMP_D, 16, &d_best));
    PM_CUDA(cudaMemsetAsync(d_best, 0xFF, sizeof(unsigned long long), c->stream));
    const uint64_t per_tile = static_cast<uint64_t>(k::kMedianThreads) * k::kMedianCands;
    const uint64_t tiles = (candidates + per_tile - 1) / per_tile;
    const unsigned grid = static_cast<unsigned>(std::min<uint64_t>(tiles, static_cast<uint64_t>(c->sm_count) * 8));
    k::median_string_kernel<<<grid, k::kMedianThreads, 0, c->stream>>>(c->d_words, c->d_word_off, c->d_seq_len, c->t, l,
                                                                      candidates, d_best);
    PM_TRY(check_launch(c, "median_string"));
    unsigned long long best = 0;
    PM_TRY(d2h(c, &best, d_best, sizeof(best)));
    PM_CUDA(cudaStreamSynchronize(c->stream));
    *total_distance = static_cast<int>(best >> 32);
    unpack_consensus((best & 0xFFFFFFFFULL) << (64 - 2 * l), l, median);
    return PM_OK;
}

// ------------------------------------------------------------------------------------------------
// run(), driver.hpp:145-220
// ------------------------------------------------------------------------------------------------
}  // extern "C"

namespace {

struct TrialSummary {  // device layout of S_TB: parallel arrays would need 6 copies; one struct, one copy
    int32_t work;      // -1 when the trial has no enriched bucket
    int32_t score;
    int32_t iters;
    int32_t n_close;   // other buckets of the trial whose score equals the best and whose expectation is within kTieEps
    double expct;
    uint64_t key;
    uint64_t cons;
};

// Expectations of the FP32 kernels agree with the reference to 1e-5 (largest difference seen over ~2.5 M refined buckets
// of C1-C4: 9e-6), so two of them can be off by 2e-5 against each other; two candidates of equal score closer than
// kTieEps are re-refined in FP64 before they are compared (the reference compares doubles exactly, driver.hpp:131-133).
constexpr double kTieEps = 5e-5;

// Per trial of the batch, one CTA: the trial's best bucket under candidate_improves (driver.hpp:127-135, :169-175:
// lexicographic (score, expectation, smaller key) -- a strict total order within a trial, keys are unique), the number
// of other buckets FP32 cannot separate from it, its summary record, its positions (gathered next to each other so that
// one copy brings the winner's along) and the XOR/popcount scan of its consensus over every window (sequence.hpp:28-38,
// oracle.hpp:101-115: total distance and the number of sequences with an occurrence within d).  With these the host
// needs one read-back per batch and no second round trip for the winner's positions or the final scoring.
__global__ void __launch_bounds__(256) trial_reduce_kernel(const unsigned int* __restrict__ work_off, const k::WorkDesc* __restrict__ work,
                                                          const int32_t* __restrict__ score, const int32_t* __restrict__ iters,
                                                          const double* __restrict__ expct, const uint64_t* __restrict__ cons,
                                                          const int32_t* __restrict__ pos, int n_trials, int t, int l, int d,
                                                          double tie_eps, const uint64_t* __restrict__ words,
                                                          const int64_t* __restrict__ word_off, const int32_t* __restrict__ seq_len,
                                                          int32_t* __restrict__ best_work, TrialSummary* __restrict__ out,
                                                          int32_t* __restrict__ pos_best, int32_t* __restrict__ ham) {
    __shared__ int s_within, s_total, s_best;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    const uint64_t digit_mask = (0x5555555555555555ULL >> (64 - 2 * l)) << (64 - 2 * l);
    for (int tr = blockIdx.x; tr < n_trials; tr += gridDim.x) {
        if (threadIdx.x == 0) {
            s_within = 0;
            s_total = 0;
        }
        if (warp == 0) {
            const unsigned int b = work_off[tr], e = work_off[tr + 1];
            int bi = -1, bs = -1;
            double be = 0.0;
            uint64_t bk = 0;
            for (unsigned int w = b + lane; w < e; w += 32) {
                const int sc = score[w];
                const double ex = expct[w];
                const uint64_t key = work[w].key;
                if (bi < 0 || k::better(sc, ex, key, bs, be, bk)) {
                    bi = static_cast<int>(w);
                    bs = sc;
                    be = ex;
                    bk = key;
                }
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
                const int os = __shfl_xor_sync(0xffffffffu, bs, o);
                const double oe = __shfl_xor_sync(0xffffffffu, be, o);
                const uint64_t ok = __shfl_xor_sync(0xffffffffu, bk, o);
                if (oi >= 0 && (bi < 0 || k::better(os, oe, ok, bs, be, bk))) {
                    bi = oi;
                    bs = os;
                    be = oe;
                    bk = ok;
                }
            }
            // candidates the FP32 expectation cannot separate from the best (driver.hpp:131-133 compares doubles exactly)
            int close = 0;
            for (unsigned int w = b + lane; w < e; w += 32) {
                if (static_cast<int>(w) != bi && score[w] == bs && fabs(expct[w] - be) <= tie_eps) ++close;
            }
            close = __reduce_add_sync(0xffffffffu, close);
            if (lane == 0) {
                s_best = bi;
                best_work[tr] = bi;
                TrialSummary sm;
                sm.work = bi;
                sm.n_close = close;
                sm.score = bi >= 0 ? bs : -1;
                sm.iters = bi >= 0 ? iters[bi] : 0;
                sm.expct = bi >= 0 ? be : 0.0;
                sm.key = bi >= 0 ? bk : 0;
                sm.cons = bi >= 0 ? cons[bi] : 0;
                out[tr] = sm;
            }
        }
        __syncthreads();
        const int w = s_best;
        if (w >= 0) {
            if (pos_best != nullptr && pos != nullptr) {
                for (int i = threadIdx.x; i < t; i += blockDim.x)
                    pos_best[static_cast<int64_t>(tr) * t + i] = pos[static_cast<int64_t>(w) * t + i];
            }
            const uint64_t cand = cons[w];
            for (int i = warp; i < t; i += nwarps) {
                const uint64_t* wp = words + word_off[i];
                const int W = seq_len[i] - l + 1;
                int best = 64;
                for (int j = lane; j < W; j += 32) {
                    const uint64_t xr = k::load_window(wp, j) ^ cand;
                    best = min(best, __popcll((xr | (xr >> 1)) & digit_mask));
                }
                best = __reduce_min_sync(0xffffffffu, best);
                if (lane == 0) {
                    atomicAdd(&s_total, best);
                    if (best <= d) atomicAdd(&s_within, 1);
                }
            }
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            ham[2 * tr] = s_within;
            ham[2 * tr + 1] = s_total;
        }
        __syncthreads();
    }
}

struct RunState {
    bool have_best = false;
    TrialSummary best{};
    int64_t best_trial = 0;
    std::vector<int32_t> positions;
    std::vector<int32_t> best_members;  // member list of the incumbent (kept so it can be re-refined in FP64 later)
    bool best_exact = false;            // best.expct is the FP64 kernel's value
    int32_t best_in_batch = -1;         // work item of the incumbent if it belongs to the batch being reduced
    int64_t exact_refines = 0;          // FP64 re-refinements this run needed
    bool ham_valid = false;             // within_d / total_distance of the incumbent came back with its batch
    int32_t within_d = 0, total_distance = 0;
};

// FP64 expectation (and score) of one member list: pm_em_f64.cuh through the stage path
int exact_candidate(pm_ctx* c, const pm_run_config* cfg, const std::vector<int32_t>& members, double* expct, int32_t* score) {
    const int64_t off[2] = {0, static_cast<int64_t>(members.size())};
    return pm_refine_exact(c, cfg->l, members.data(), off, 1, cfg->max_em_iters, cfg->em_tol, nullptr, nullptr, score, expct,
                           nullptr, nullptr, nullptr);
}

// member list of work item w of the current batch
int fetch_members(pm_ctx* c, const k::WorkDesc* d_work, const unsigned int* d_members, int32_t w, std::vector<int32_t>* out,
                  k::WorkDesc* wd_out) {
    k::WorkDesc wd;
    PM_TRY(d2h(c, &wd, d_work + w, sizeof(wd)));
    PM_CUDA(cudaStreamSynchronize(c->stream));
    out->resize(wd.count);
    PM_TRY(d2h(c, out->data(), d_members + wd.mem_begin, sizeof(int32_t) * wd.count));
    PM_CUDA(cudaStreamSynchronize(c->stream));
    if (wd_out) *wd_out = wd;
    return PM_OK;
}

// must mirror the carve-up at the top of hash_bucket_fused_kernel
size_t fused_hash_smem_bytes(int n_words, int keybits, int64_t cap_e, int t, int64_t x) {
    const size_t n_keys = static_cast<size_t>(1) << keybits;
    size_t b = static_cast<size_t>(n_words) * 8 + n_keys * 2 + std::max<size_t>(n_keys / 32, 1) * 4;
    b += static_cast<size_t>(cap_e) * 4 + (2 * static_cast<size_t>(t) + 1) * 4 + (2 * (k::kFusedThreads / 32) + 2) * 4;
    b += static_cast<size_t>(x) * 2 + 8 + 8;
    return b + 16;
}

bool fused_hash_applies(const pm_ctx* c, int keybits, int64_t cap_e) {
    const char* env = std::getenv("PM_B200_FUSED_HASH");  // test/tuning knob: 0 selects the radix-sort path
    if (env != nullptr && std::atoi(env) == 0) return false;
    return keybits <= 16 && c->x < 65536 && c->total_words <= k::kPairMaxWords &&
           fused_hash_smem_bytes(static_cast<int>(c->total_words), keybits, cap_e, c->t, c->x) <= 200 * 1024;
}

// hash_trial + enriched_buckets of every trial of the batch, one CTA per trial (pm_hash_fused.cuh)
// plans of trials first, first + stride, ... sampled on the device (pm_plans.cuh) into S_PLANS; *fail (device) is
// raised when a trial needed more PRNG outputs than the sampler holds
int sample_plans_on_device(pm_ctx* c, int l, int kk, uint64_t master, int64_t first, int64_t stride, int n, k::PlanProg** d_progs,
                           int32_t* d_kept, unsigned int** d_fail) {
    unsigned char* raw;
    PM_TRY(get_buf(c, S_PLANS, sizeof(k::PlanProg) * static_cast<size_t>(n) + 16, &raw));
    *d_fail = reinterpret_cast<unsigned int*>(raw);
    *d_progs = reinterpret_cast<k::PlanProg*>(raw + 16);
    PM_CUDA(cudaMemsetAsync(*d_fail, 0, sizeof(unsigned int), c->stream));
    k::plan_sample_kernel<<<(n + 63) / 64, 64, 0, c->stream>>>(master, first, stride, n, l, kk, *d_progs, d_kept, *d_fail);
    return check_launch(c, "plan_sample");
}

int fused_hash_bucket(pm_ctx* c, const std::vector<k::PlanProg>& progs, int keybits, int thr, unsigned int* members,
                      Records* r, const k::PlanProg* d_progs = nullptr) {
    r->cap_e = std::max<int64_t>(1, c->x / thr);
    const int n = static_cast<int>(progs.size());
    const size_t nrec = static_cast<size_t>(n) * static_cast<size_t>(r->cap_e);
    PM_TRY(get_buf(c, S_REC_KEY, nrec, &r->key));
    PM_TRY(get_buf(c, S_REC_START, nrec, &r->start));
    PM_TRY(get_buf(c, S_REC_SIZE, nrec, &r->size));
    PM_TRY(get_buf(c, S_NREC, static_cast<size_t>(n) + 1, &r->n_rec));
    const size_t smem = fused_hash_smem_bytes(static_cast<int>(c->total_words), keybits, r->cap_e, c->t, c->x);
    PM_TRY(ensure_dynamic_smem(reinterpret_cast<const void*>(k::hash_bucket_fused_kernel), smem, false));
    k::FusedHashParams p;
    p.words = c->d_words;
    p.word_off = c->d_word_off;
    p.win_off = c->d_win_off;
    p.t = c->t;
    p.keybits = keybits;
    p.x = static_cast<int>(c->x);
    p.n_words = static_cast<int>(c->total_words);
    p.thr = thr;
    p.cap_e = static_cast<int>(r->cap_e);
    p.members = members;
    p.rec_key = r->key;
    p.rec_start = r->start;
    p.rec_size = r->size;
    p.n_rec = r->n_rec;
    for (int base = 0; base < n; base += k::kMaxConstPlans) {
        const int cnt = std::min(k::kMaxConstPlans, n - base);
        if (d_progs == nullptr) c->h2d_bytes += static_cast<int64_t>(sizeof(k::PlanProg)) * cnt;
        ConstPlansUse plans_use(c->device, c->stream);
        if (d_progs != nullptr) {
            PM_CUDA(cudaMemcpyToSymbolAsync(k::c_plans, d_progs + base, sizeof(k::PlanProg) * static_cast<size_t>(cnt), 0,
                                            cudaMemcpyDeviceToDevice, c->stream));
        } else {
            PM_CUDA(cudaMemcpyToSymbolAsync(k::c_plans, progs.data() + base, sizeof(k::PlanProg) * static_cast<size_t>(cnt),
                                            0, cudaMemcpyHostToDevice, c->stream));
        }
        p.plan_base = base;
        p.n_trials = cnt;
        const unsigned grid = static_cast<unsigned>(std::min(cnt, 2 * c->sm_count));
        k::hash_bucket_fused_kernel<<<grid, k::kFusedThreads, smem, c->stream>>>(p);
        PM_TRY(check_launch(c, "hash_bucket_fused"));
    }
    return PM_OK;
}

// Large sets with a dense table of at most 2^20 entries: device-wide counting sort (pm_hash_count.cuh) -- when the
// mean bucket size x / 4^k is below the threshold s, i.e. when enriched buckets are the exception (10,000 sequences,
// k = 10, s = 19: 1 % of the l-mers are members).  When nearly every l-mer is a member of an enriched bucket (the same
// set with k = 7, s = 4: 16,384 buckets of ~600) the contended cursor atomics and the per-bucket ordering cost more
// than the three passes of the radix sort (measured 0.85 against 0.69 ms per trial), so that stays on the sort path.
// PM_B200_COUNT_HASH: 0 never, 2 whenever the table fits (tests).
bool count_hash_applies(const pm_ctx* c, int keybits, int thr) {
    const char* env = std::getenv("PM_B200_COUNT_HASH");
    const int mode = env != nullptr ? std::atoi(env) : 1;
    if (mode == 0 || keybits > 20) return false;
    return mode >= 2 || c->x < static_cast<int64_t>(thr) * (1LL << keybits);
}

// hash_trial + enriched_buckets of every trial of the batch.  *ok = false when some enriched bucket is too large for
// the in-CTA ordering step (degenerate input): the caller then takes the radix-sort path.  One host sync per batch
// (the size check) -- on this path a trial's EM stage takes seconds.
int count_hash_bucket(pm_ctx* c, const std::vector<k::PlanProg>& progs, int keybits, int thr, unsigned int** members,
                      Records* r, bool* ok) {
    const int n = static_cast<int>(progs.size());
    const int64_t tsize = 1LL << keybits;
    r->cap_e = std::max<int64_t>(1, c->x / thr);
    const size_t nrec = static_cast<size_t>(n) * static_cast<size_t>(r->cap_e);
    PM_TRY(get_buf(c, S_REC_KEY, nrec, &r->key));
    PM_TRY(get_buf(c, S_REC_START, nrec, &r->start));
    PM_TRY(get_buf(c, S_REC_SIZE, nrec, &r->size));
    PM_TRY(get_buf(c, S_NREC, static_cast<size_t>(n), &r->n_rec));
    unsigned int* table;
    unsigned int* slots;
    const size_t table_words = static_cast<size_t>(n) * static_cast<size_t>(tsize);
    PM_TRY(get_buf(c, S_COUNTS, table_words + 1, &table));  // + the largest enriched bucket of the batch
    PM_TRY(get_buf(c, S_IDX_A, static_cast<size_t>(n) * static_cast<size_t>(c->x), &slots));
    unsigned int* d_max = table + table_words;
    PM_CUDA(cudaMemsetAsync(table, 0, (table_words + 1) * sizeof(unsigned int), c->stream));
    k::CountParams p;
    p.words = c->d_words;
    p.word_off = c->d_word_off;
    p.win_off = c->d_win_off;
    p.t = c->t;
    p.x = c->x;
    p.uniform_w = c->uniform_w;
    p.table_size = tsize;
    p.table = table;
    const unsigned gx = static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>((c->x + 255) / 256, 8LL * c->sm_count)));
    for (int base = 0; base < n; base += k::kMaxConstPlans) {
        const int cnt = std::min(k::kMaxConstPlans, n - base);
        c->h2d_bytes += static_cast<int64_t>(sizeof(k::PlanProg)) * cnt;
        ConstPlansUse plans_use(c->device, c->stream);
        PM_CUDA(cudaMemcpyToSymbolAsync(k::c_plans, progs.data() + base, sizeof(k::PlanProg) * static_cast<size_t>(cnt),
                                        0, cudaMemcpyHostToDevice, c->stream));
        p.plan_base = base;
        p.n_trials = cnt;
        const dim3 grid(gx, static_cast<unsigned>(std::min(cnt, 64)));
        k::count_hist_kernel<<<grid, 256, 0, c->stream>>>(p);
        PM_TRY(check_launch(c, "count_hist"));
        const int n_chunks = static_cast<int>((tsize + k::kCountChunk - 1) / k::kCountChunk);
        uint2* partial;
        PM_TRY(get_buf(c, S_DIGIT_TOT, static_cast<size_t>(cnt) * static_cast<size_t>(n_chunks), &partial));
        const dim3 sgrid(static_cast<unsigned>(n_chunks), static_cast<unsigned>(cnt));
        k::count_partial_kernel<<<sgrid, k::kCountScanThreads, 0, c->stream>>>(
            table + static_cast<size_t>(base) * static_cast<size_t>(tsize), tsize, thr, n_chunks, partial);
        PM_TRY(check_launch(c, "count_partial"));
        k::count_scan_kernel<<<sgrid, k::kCountScanThreads, 0, c->stream>>>(
            table + static_cast<size_t>(base) * static_cast<size_t>(tsize), tsize, thr, r->cap_e, n_chunks, partial,
            r->key + static_cast<size_t>(base) * static_cast<size_t>(r->cap_e),
            r->start + static_cast<size_t>(base) * static_cast<size_t>(r->cap_e),
            r->size + static_cast<size_t>(base) * static_cast<size_t>(r->cap_e), r->n_rec + base, d_max);
        PM_TRY(check_launch(c, "count_scan"));
        k::count_scatter_kernel<<<grid, 256, 0, c->stream>>>(p, slots);
        PM_TRY(check_launch(c, "count_scatter"));
    }
    unsigned int h_max = 0;
    PM_TRY(d2h(c, &h_max, d_max, sizeof(h_max)));
    PM_CUDA(cudaStreamSynchronize(c->stream));
    *ok = h_max <= static_cast<unsigned int>(k::kCountMaxBucket);
    if (!*ok) return PM_OK;
    const unsigned ox = static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(r->cap_e, 16LL * c->sm_count)));
    k::count_order_kernel<<<dim3(ox, static_cast<unsigned>(std::min(n, 64))), k::kCountOrderThreads, 0, c->stream>>>(
        slots, c->x, r->cap_e, n, r->start, r->size, r->n_rec);
    PM_TRY(check_launch(c, "count_order"));
    *members = slots;
    return PM_OK;
}

constexpr int kRetryWithHostPlans = -77;  // internal to pm_run / run_batch

template <typename KeyT>
int run_batch(pm_ctx* c, const pm_run_config* cfg, const pm_run_result& params, const std::vector<k::PlanProg>& progs,
              int64_t first_trial, pm_run_result* out, RunState* st, bool* stop, int64_t* trial_buckets,
              int32_t* trial_best_score, double* trial_best_expectation, uint64_t* trial_best_key, int64_t out_base,
              bool more_batches, int64_t trial_stride, bool device_plans) {
    const int n_trials = static_cast<int>(progs.size());
    st->best_in_batch = -1;
    const int l = cfg->l;
    const bool prof = cfg->profile != 0;
    const int r_cap = c->t * params.s;
    Sorted<KeyT> srt;
    Records rec;
    const bool fused = fused_hash_applies(c, 2 * params.k, std::max<int64_t>(1, c->x / params.s));
    unsigned int* d_plan_fail = nullptr;
    if (device_plans && !fused) return set_error(PM_ERR_CUDA, "internal: device plans without the one-CTA bucketing");
    if (fused) {
        StageTimer tk(c, prof, 0);
        PM_TRY(get_buf(c, S_IDX_A, progs.size() * static_cast<size_t>(c->x), &srt.idx));
        k::PlanProg* d_progs = nullptr;
        if (device_plans)  // the reference's PRNG stream, one thread per trial (pm_plans.cuh): nothing to sample or upload here
            PM_TRY(sample_plans_on_device(c, l, params.k, cfg->seed, first_trial, trial_stride, n_trials, &d_progs, nullptr, &d_plan_fail));
        PM_TRY(fused_hash_bucket(c, progs, 2 * params.k, params.s, srt.idx, &rec, d_progs));
    }
    bool counted = false;
    if (!fused && count_hash_applies(c, 2 * params.k, params.s)) {
        StageTimer tk(c, prof, 0);
        PM_TRY(count_hash_bucket(c, progs, 2 * params.k, params.s, &srt.idx, &rec, &counted));
    }
    if (!fused && !counted) {
        StageTimer tk(c, prof, 0);
        const size_t n = progs.size() * static_cast<size_t>(c->x);
        KeyT *ka, *kb;
        unsigned int *ia, *ib;
        PM_TRY(get_buf(c, S_KEYS_A, n, &ka));
        PM_TRY(get_buf(c, S_KEYS_B, n, &kb));
        PM_TRY(get_buf(c, S_IDX_A, n, &ia));
        PM_TRY(get_buf(c, S_IDX_B, n, &ib));
        PM_TRY(project_keys<KeyT>(c, progs, ka));
        tk.stop();
        StageTimer ts(c, prof, 1);
        PM_TRY((sort_segments<KeyT>(c, ka, kb, ia, ib, n_trials, c->x, c->x, nullptr, 2 * params.k, &srt.keys, &srt.idx)));
    }
    unsigned int* work_off;
    k::WorkDesc* work;
    {
        StageTimer te(c, prof, 2);
        if (!fused && !counted) PM_TRY(find_enriched<KeyT>(c, srt, n_trials, params.s, &rec));
        PM_TRY(get_buf(c, S_WORK_OFF, static_cast<size_t>(n_trials) + 1, &work_off));
        PM_TRY(get_buf(c, S_WORK, static_cast<size_t>(n_trials) * static_cast<size_t>(rec.cap_e), &work));
        k::work_scan_kernel<<<1, 1024, 0, c->stream>>>(rec.n_rec, n_trials, work_off);
        PM_TRY(check_launch(c, "work_scan"));
        const unsigned gx = static_cast<unsigned>(std::min<int64_t>((rec.cap_e + 127) / 128, 64));
        k::build_work_kernel<<<dim3(std::max(gx, 1u), static_cast<unsigned>(n_trials)), 128, 0, c->stream>>>(
            rec.n_rec, work_off, rec.key, rec.start, rec.size, c->x, rec.cap_e, r_cap, n_trials, work);
        PM_TRY(check_launch(c, "build_work"));
    }
    const size_t nb = static_cast<size_t>(n_trials) * static_cast<size_t>(rec.cap_e);
    EmOut o;
    unsigned long long* d_scal;
    int32_t* best_work;
    TrialSummary* d_tb;
    PM_TRY(get_buf(c, S_OUT_SCORE, nb, &o.score));
    PM_TRY(get_buf(c, S_OUT_ITERS, nb, &o.iters));
    PM_TRY(get_buf(c, S_OUT_EXP, nb, &o.expct));
    PM_TRY(get_buf(c, S_OUT_CONS, nb, &o.cons));
    // positions of every bucket are written by the main launch when that is affordable; otherwise the
    // winning bucket is re-run alone afterwards (deterministic kernel => identical candidate)
    const bool all_positions = nb * static_cast<size_t>(c->t) * sizeof(int32_t) <= (256u << 20);
    if (all_positions) PM_TRY(get_buf(c, S_OUT_POS, nb * static_cast<size_t>(c->t), &o.pos));
    PM_TRY(get_buf(c, S_SCAL, 16, &d_scal));
    PM_TRY(get_buf(c, S_BEST, static_cast<size_t>(n_trials), &best_work));
    PM_TRY(get_buf(c, S_TB, static_cast<size_t>(n_trials), &d_tb));
    PM_CUDA(cudaMemsetAsync(d_scal, 0, sizeof(unsigned long long) * 16, c->stream));
    {
        StageTimer tm(c, prof, 3);
        PM_TRY(launch_em(c, l, cfg->max_em_iters, cfg->em_tol, cfg->z_epsilon, work, work_off + n_trials, 0,
                         static_cast<unsigned int>(std::min<size_t>(nb, 1u << 30)), srt.idx, o, d_scal, r_cap));
    }
    host_mark("launched");
    std::vector<TrialSummary> tb(static_cast<size_t>(n_trials));
    std::vector<unsigned int> n_rec(static_cast<size_t>(n_trials));
    unsigned long long scal[16] = {0};
    // per-trial reduction (trial_reduce_kernel); everything the host needs from this batch comes back through one
    // pinned staging area behind a single synchronisation
    const bool epi_pos = all_positions && static_cast<size_t>(n_trials) * static_cast<size_t>(c->t) * sizeof(int32_t) <= (8u << 20);
    auto up16 = [](size_t v) { return (v + 15) & ~static_cast<size_t>(15); };
    const size_t off_tb = 0, off_nrec = up16(off_tb + sizeof(TrialSummary) * tb.size()),
                 off_scal = up16(off_nrec + sizeof(unsigned int) * n_rec.size()), off_ham = up16(off_scal + sizeof(scal)),
                 off_fail = up16(off_ham + sizeof(int32_t) * 2 * static_cast<size_t>(n_trials)), off_pos = up16(off_fail + 16),
                 pin_bytes = off_pos + (epi_pos ? sizeof(int32_t) * static_cast<size_t>(n_trials) * static_cast<size_t>(c->t) : 0);
    unsigned char* pin;
    PM_TRY(get_pinned(c, pin_bytes, reinterpret_cast<void**>(&pin)));
    const int32_t* ham = reinterpret_cast<const int32_t*>(pin + off_ham);
    const int32_t* pos_best = reinterpret_cast<const int32_t*>(pin + off_pos);
    {
        StageTimer ts4(c, prof, 4);
        int32_t* d_pos_best = nullptr;
        int32_t* d_ham;
        if (epi_pos) PM_TRY(get_buf(c, S_POS_BEST, static_cast<size_t>(n_trials) * static_cast<size_t>(c->t), &d_pos_best));
        PM_TRY(get_buf(c, S_HAM, static_cast<size_t>(n_trials) * 2, &d_ham));
        trial_reduce_kernel<<<static_cast<unsigned>(std::min(n_trials, 8 * c->sm_count)), 256, 0, c->stream>>>(
            work_off, work, o.score, o.iters, o.expct, o.cons, epi_pos ? o.pos : nullptr, n_trials, c->t, l, cfg->d, kTieEps,
            c->d_words, c->d_word_off, c->d_seq_len, best_work, d_tb, d_pos_best, d_ham);
        PM_TRY(check_launch(c, "trial_reduce"));
        ts4.stop();
        StageTimer td(c, prof, 7);
        if (epi_pos) PM_TRY(d2h(c, pin + off_pos, d_pos_best, sizeof(int32_t) * static_cast<size_t>(n_trials) * static_cast<size_t>(c->t)));
        PM_TRY(d2h(c, pin + off_ham, d_ham, sizeof(int32_t) * 2 * static_cast<size_t>(n_trials)));
        PM_TRY(d2h(c, pin + off_tb, d_tb, sizeof(TrialSummary) * tb.size()));
        PM_TRY(d2h(c, pin + off_nrec, rec.n_rec, sizeof(unsigned int) * n_rec.size()));
        PM_TRY(d2h(c, pin + off_scal, d_scal, sizeof(scal)));
        if (d_plan_fail != nullptr) PM_TRY(d2h(c, pin + off_fail, d_plan_fail, sizeof(unsigned int)));
        td.stop();
        PM_CUDA(cudaStreamSynchronize(c->stream));
        // a trial needed more PRNG outputs than the device sampler holds (probability ~1e-17 per trial): nothing of this
        // batch has been consumed yet, the caller samples its plans on the host and runs it again
        if (d_plan_fail != nullptr && *reinterpret_cast<const unsigned int*>(pin + off_fail) != 0) return kRetryWithHostPlans;
        std::memcpy(tb.data(), pin + off_tb, sizeof(TrialSummary) * tb.size());
        std::memcpy(n_rec.data(), pin + off_nrec, sizeof(unsigned int) * n_rec.size());
        std::memcpy(scal, pin + off_scal, sizeof(scal));
    }
    host_mark("gpu-wait");
    std::vector<int32_t> tb_dev_work(static_cast<size_t>(n_trials));
    for (int i = 0; i < n_trials; ++i) tb_dev_work[static_cast<size_t>(i)] = tb[static_cast<size_t>(i)].work;
    collect_stage_times(c, out->stage_ms);
#ifdef PM_TC_TIMING
    std::fprintf(stderr, "[tc clocks, CTA 0 softmax thread] total %llu  wait S %llu  wait O %llu  updates %llu | EM passes %llu  MAX passes %llu  final %llu | sequence close %llu\n",
                 scal[8], scal[9], scal[10], scal[11], scal[12], scal[13], scal[14], scal[15]);
#endif
#ifdef PM_EM_TIMING
    {
        unsigned long long tot = 0;
        for (int i = 8; i < 16; ++i) tot += scal[i];
        std::fprintf(stderr, "[em phases] init %.1f%% tables %.1f%% estep %.1f%% mstep %.1f%% update %.1f%% final %.1f%% out %.1f%% (total %.3g clk)\n",
                     100.0 * scal[8] / tot, 100.0 * scal[9] / tot, 100.0 * scal[10] / tot, 100.0 * scal[11] / tot,
                     100.0 * scal[12] / tot, 100.0 * scal[13] / tot, 100.0 * scal[14] / tot, static_cast<double>(tot));
    }
#endif
    if ((scal[1] & 0xFFFFFFFFULL) != 0) {
        return set_error(PM_ERR_NUMERICAL_UNDERFLOW, "all window weights vanished in some sequence");
    }
    const bool tc_bypassed = (scal[4] | scal[5] | scal[6] | scal[7]) == 0 && (scal[3] & 0xFFFFFFFFULL) != 0;
    if (tc_bypassed) {  // a small batch handed over wholesale: not "refined again", and no tensor work
        scal[3] = 0;
        c->tc_used = false;
    }
    c->em_exact[0] += static_cast<int64_t>(scal[3] & 0xFFFFFFFFULL);
    for (int r = 0; r < 4; ++r) c->em_exact[1 + r] += static_cast<int64_t>(scal[4 + r]);
    c->em_exact[5] += static_cast<int64_t>(scal[2] & 0xFFFFFFFFULL);
    out->em_exact_buckets += static_cast<int64_t>(scal[3] & 0xFFFFFFFFULL);
    out->em_fp64_buckets += static_cast<int64_t>(scal[2] & 0xFFFFFFFFULL);
    out->em_lookup_adds += static_cast<int64_t>(scal[0]) * c->x * l;
    {
        // W_EM = sum_b (2 I_b + 1) x l lookup-adds + 4 (I_b + 1) x; scal[0] = sum_b (I_b + 1)
        int64_t n_buckets = 0;
        for (unsigned int nr : n_rec) n_buckets += nr;
        const int64_t s_iters1 = static_cast<int64_t>(scal[0]);
        out->em_work += (2 * s_iters1 - n_buckets) * c->x * l + 4 * s_iters1 * c->x;
        if (c->tc_used) {
            // passes of a tile (pm_em_tc.cuh): I EM passes and the final E-step with three log-odds terms; GEMM2 in the
            // I EM passes
            const int64_t I = cfg->max_em_iters, tiles = (n_buckets + k::kTcRows - 1) / k::kTcRows;
            out->em_tensor_flops += tiles * (c->tc_g1_flops * 3 * (I + 1) + c->tc_g2_flops * I);
        }
    }

    // Trials whose best bucket the FP32 expectation cannot separate from another bucket of the same score: every such
    // candidate is refined again in FP64 and the comparison of driver.hpp:172-174 is repeated on those values.
    // All such trials of the batch are settled together: their candidates go through ONE FP64 launch and the copies that
    // gather them share a handful of synchronisations (a trial at a time cost ~0.6 ms each on the n = 1000 sets).
    std::vector<char> tb_exact(static_cast<size_t>(n_trials), 0);
    {
        // Only a trial that can still become the incumbent needs it: in the ascending scan below the incumbent's score is
        // the largest score seen so far, so a trial scoring less cannot improve on it whatever its expectation (its
        // per-trial record is settled only when the caller asked for per-trial outputs).
        const bool want_all = trial_best_score != nullptr || trial_best_expectation != nullptr || trial_best_key != nullptr;
        int run_max = st->have_best ? st->best.score : -1;
        std::vector<int> need;
        for (int i = 0; i < n_trials; ++i) {
            const TrialSummary& s = tb[static_cast<size_t>(i)];
            if (s.work < 0) continue;
            if (s.n_close != 0 && (want_all || s.score >= run_max)) need.push_back(i);
            run_max = std::max(run_max, s.score);
        }
        if (!need.empty()) {
            std::vector<unsigned int> woff(static_cast<size_t>(n_trials) + 1);
            PM_TRY(d2h(c, woff.data(), work_off, sizeof(unsigned int) * woff.size()));
            PM_CUDA(cudaStreamSynchronize(c->stream));
            // scores and expectations of every bucket of those trials
            std::vector<size_t> at(need.size() + 1, 0);
            for (size_t q = 0; q < need.size(); ++q)
                at[q + 1] = at[q] + (woff[static_cast<size_t>(need[q]) + 1] - woff[static_cast<size_t>(need[q])]);
            std::vector<int32_t> sc(at.back());
            std::vector<double> ex(at.back());
            for (size_t q = 0; q < need.size(); ++q) {
                const unsigned int b = woff[static_cast<size_t>(need[q])], n_b = woff[static_cast<size_t>(need[q]) + 1] - b;
                if (n_b == 0) continue;
                PM_TRY(d2h(c, sc.data() + at[q], o.score + b, sizeof(int32_t) * n_b));
                PM_TRY(d2h(c, ex.data() + at[q], o.expct + b, sizeof(double) * n_b));
            }
            PM_CUDA(cudaStreamSynchronize(c->stream));
            // every candidate of a trial that the FP32 expectation cannot separate from its best
            std::vector<int32_t> cand;               // work items
            std::vector<size_t> cand_at(need.size() + 1, 0);
            for (size_t q = 0; q < need.size(); ++q) {
                const TrialSummary& s = tb[static_cast<size_t>(need[q])];
                const unsigned int b = woff[static_cast<size_t>(need[q])];
                for (size_t w = at[q]; w < at[q + 1]; ++w) {
                    if (sc[w] != s.score || std::fabs(ex[w] - s.expct) > 2.0 * kTieEps) continue;
                    cand.push_back(static_cast<int32_t>(b + (w - at[q])));
                }
                cand_at[q + 1] = cand.size();
            }
            std::vector<k::WorkDesc> wds(cand.size());
            for (size_t q = 0; q < cand.size(); ++q) PM_TRY(d2h(c, &wds[q], work + cand[q], sizeof(k::WorkDesc)));
            PM_CUDA(cudaStreamSynchronize(c->stream));
            std::vector<int64_t> moff(cand.size() + 1, 0);
            for (size_t q = 0; q < cand.size(); ++q) moff[q + 1] = moff[q] + wds[q].count;
            std::vector<int32_t> all_members(static_cast<size_t>(moff.back()));
            for (size_t q = 0; q < cand.size(); ++q) {
                if (wds[q].count == 0) continue;
                PM_TRY(d2h(c, all_members.data() + moff[q], srt.idx + wds[q].mem_begin, sizeof(int32_t) * wds[q].count));
            }
            PM_CUDA(cudaStreamSynchronize(c->stream));
            std::vector<double> e64(cand.size());
            if (!cand.empty()) {
                PM_TRY(pm_refine_exact(c, cfg->l, all_members.data(), moff.data(), static_cast<int>(cand.size()), cfg->max_em_iters,
                                       cfg->em_tol, nullptr, nullptr, nullptr, e64.data(), nullptr, nullptr, nullptr));
                st->exact_refines += static_cast<int64_t>(cand.size());
            }
            bool moved = false;
            for (size_t q = 0; q < need.size(); ++q) {
                TrialSummary& s = tb[static_cast<size_t>(need[q])];
                bool have = false;
                int32_t bw = -1;
                double be = 0.0;
                uint64_t bk = 0;
                for (size_t r = cand_at[q]; r < cand_at[q + 1]; ++r) {
                    if (!have || pm_candidate_improves(s.score, e64[r], wds[r].key, s.score, be, bk)) {
                        have = true;
                        bw = cand[r];
                        be = e64[r];
                        bk = wds[r].key;
                    }
                }
                if (!have) continue;
                if (bw != s.work) {
                    PM_TRY(d2h(c, &s.iters, o.iters + bw, sizeof(int32_t)));
                    PM_TRY(d2h(c, &s.cons, o.cons + bw, sizeof(uint64_t)));
                    moved = true;
                }
                s.work = bw;
                s.expct = be;
                s.key = bk;
                tb_exact[static_cast<size_t>(need[q])] = 1;
            }
            if (moved) PM_CUDA(cudaStreamSynchronize(c->stream));
        }
    }

    // Ascending-trial reduction, driver.hpp:195-208.
    const int perfect = l * c->t;
    int32_t new_best_work = -1;
    int new_best_trial_idx = -1;  // index within the batch
    std::vector<int32_t> dev_work(static_cast<size_t>(n_trials));  // the device's choice per trial (the FP64 settlement above may have moved s.work)
    for (int i = 0; i < n_trials; ++i) dev_work[static_cast<size_t>(i)] = tb_dev_work[static_cast<size_t>(i)];
    for (int i = 0; i < n_trials; ++i) {
        const int64_t trial = first_trial + i * trial_stride;
        TrialSummary& s = tb[static_cast<size_t>(i)];
        out->trials_run = trial;
        out->buckets_enriched += n_rec[static_cast<size_t>(i)];
        const size_t oi = static_cast<size_t>(out_base + i);
        if (trial_buckets) trial_buckets[oi] = n_rec[static_cast<size_t>(i)];
        if (trial_best_score) trial_best_score[oi] = s.score;
        if (trial_best_expectation) trial_best_expectation[oi] = s.expct;
        if (trial_best_key) trial_best_key[oi] = s.key;
        bool improves = false;
        if (s.work >= 0) {
            if (!st->have_best) {
                improves = true;
            } else if (s.score == st->best.score && std::fabs(s.expct - st->best.expct) <= kTieEps &&
                       (s.expct != st->best.expct || static_cast<double>(static_cast<float>(s.expct)) == s.expct)) {
                // equal score, expectations closer than the FP32 error: both in FP64.  Bit-equal FP64 expectations are the
                // same model -- identical member lists -- and stay an exact tie; bit-equal values that are FP32 numbers
                // come from the tensor-core kernel, which rounds its expectation to FP32: different models can collide
                // there (two saturated models 3e-14 apart in the reference), so those are settled too.
                bool s_exact = tb_exact[static_cast<size_t>(i)] != 0;
                if (!s_exact) {
                    std::vector<int32_t> mem;
                    int32_t s64 = 0;
                    PM_TRY(fetch_members(c, work, srt.idx, s.work, &mem, nullptr));
                    PM_TRY(exact_candidate(c, cfg, mem, &s.expct, &s64));
                    ++st->exact_refines;
                    tb_exact[static_cast<size_t>(i)] = 1;
                    if (trial_best_expectation) trial_best_expectation[oi] = s.expct;
                }
                if (!st->best_exact) {
                    int32_t s64 = 0;
                    if (st->best_in_batch >= 0) PM_TRY(fetch_members(c, work, srt.idx, st->best_in_batch, &st->best_members, nullptr));
                    PM_TRY(exact_candidate(c, cfg, st->best_members, &st->best.expct, &s64));
                    ++st->exact_refines;
                    st->best_exact = true;
                }
                improves = pm_candidate_improves(s.score, s.expct, s.key, st->best.score, st->best.expct, st->best.key) != 0;
            } else {
                improves = pm_candidate_improves(s.score, s.expct, s.key, st->best.score, st->best.expct, st->best.key) != 0;
            }
        }
        if (improves) {
            st->have_best = true;
            st->best = s;
            st->best_trial = trial;
            st->best_exact = tb_exact[static_cast<size_t>(i)] != 0;
            st->best_in_batch = s.work;
            new_best_work = s.work;
            new_best_trial_idx = i;
        }
        if (cfg->early_stop && st->have_best && st->best.score == perfect) {
            *stop = true;
            break;
        }
    }
    // a later batch may have to re-refine the incumbent in FP64: keep its member list (this batch's buffers are reused)
    if (more_batches && st->best_in_batch >= 0) PM_TRY(fetch_members(c, work, srt.idx, st->best_in_batch, &st->best_members, nullptr));
    st->best_in_batch = -1;
    const bool epi_hit = new_best_work >= 0 && dev_work[static_cast<size_t>(new_best_trial_idx)] == new_best_work;
    if (new_best_work >= 0) {
        st->ham_valid = epi_hit;
        if (epi_hit) {
            st->within_d = ham[2 * static_cast<size_t>(new_best_trial_idx)];
            st->total_distance = ham[2 * static_cast<size_t>(new_best_trial_idx) + 1];
        }
    }
    if (epi_hit && epi_pos) {
        // the winner's positions came back with the summaries
        st->positions.assign(pos_best + static_cast<int64_t>(new_best_trial_idx) * c->t,
                             pos_best + static_cast<int64_t>(new_best_trial_idx + 1) * c->t);
    } else if (new_best_work >= 0 && all_positions) {
        st->positions.resize(static_cast<size_t>(c->t));
        PM_TRY(d2h(c, st->positions.data(), o.pos + static_cast<size_t>(new_best_work) * static_cast<size_t>(c->t),
                   sizeof(int32_t) * static_cast<size_t>(c->t)));
        PM_CUDA(cudaStreamSynchronize(c->stream));
    } else if (new_best_work >= 0) {
        // Positions of the new incumbent: re-run its bucket alone with the position output on.
        // Same kernel, same launch shape per CTA, deterministic => identical candidate.
        EmOut o1;
        PM_TRY(get_buf(c, S_TMP_A, 16, &o1.score));
        o1.iters = o1.score + 4;
        PM_TRY(get_buf(c, S_TMP_B, 4, &o1.expct));
        PM_TRY(get_buf(c, S_TMP_C, 4, &o1.cons));
        PM_TRY(get_buf(c, S_OUT_POS, static_cast<size_t>(c->t), &o1.pos));
        unsigned long long* d_scal2;
        PM_TRY(get_buf(c, S_TMP_D, 16, &d_scal2));
        PM_CUDA(cudaMemsetAsync(d_scal2, 0, sizeof(unsigned long long) * 16, c->stream));
        PM_TRY(launch_em(c, l, cfg->max_em_iters, cfg->em_tol, cfg->z_epsilon, work + new_best_work, nullptr, 1, 1, srt.idx,
                         o1, d_scal2));
        st->positions.resize(static_cast<size_t>(c->t));
        PM_TRY(d2h(c, st->positions.data(), o1.pos, sizeof(int32_t) * static_cast<size_t>(c->t)));
        PM_CUDA(cudaStreamSynchronize(c->stream));
    }
    return PM_OK;
}

}  // namespace

extern "C" {

int pm_ctx_trial_plans(pm_ctx* c, int l, int k, uint64_t master, int64_t first_trial, int64_t stride, int n, int32_t* kept) {
    clear_error();
    if (c == nullptr || kept == nullptr) return set_error(PM_ERR_INVALID_PARAMS, "null argument");
    if (l < 1 || l > 31 || k < 1 || k > l || n < 1 || stride < 1 || first_trial < 1)
        return set_error(PM_ERR_INVALID_PARAMS, "device plans need 1 <= k <= l <= 31, n >= 1, stride >= 1, first_trial >= 1");
    PM_CUDA(cudaSetDevice(c->device));
    int32_t* d_kept;
    PM_TRY(get_buf(c, S_PLAN_KEPT, static_cast<size_t>(n) * static_cast<size_t>(k), &d_kept));
    k::PlanProg* d_progs;
    unsigned int* d_fail;
    PM_TRY(sample_plans_on_device(c, l, k, master, first_trial, stride, n, &d_progs, d_kept, &d_fail));
    unsigned int fail = 0;
    PM_TRY(d2h(c, kept, d_kept, sizeof(int32_t) * static_cast<size_t>(n) * static_cast<size_t>(k)));
    PM_TRY(d2h(c, &fail, d_fail, sizeof(fail)));
    PM_CUDA(cudaStreamSynchronize(c->stream));
    if (fail != 0) return set_error(PM_ERR_UNSUPPORTED, "a trial needed more PRNG outputs than the device sampler holds");
    return PM_OK;
}

int pm_run(pm_ctx* c, const pm_run_config* cfg, pm_run_result* out, int32_t* positions, int64_t* trial_buckets,
           int32_t* trial_best_score, double* trial_best_expectation, uint64_t* trial_best_key) {
    const auto t0 = std::chrono::steady_clock::now();
    clear_error();
    if (cfg == nullptr || out == nullptr) return set_error(PM_ERR_INVALID_PARAMS, "null argument");
    PM_TRY(need_sequences(c));
    std::memset(out, 0, sizeof(*out));
    PM_TRY(pm_resolve_params(cfg, c->offs.data(), c->t, out));
    const pm_run_result params = *out;
    PM_TRY(prepare_windows(c, cfg->l));
    if (params.k > 31) {
        return set_error(PM_ERR_KMER_TOO_LONG, "projection width " + std::to_string(params.k) +
                                                   " exceeds the encodable k-mer length 31");
    }
    PM_TRY(check_backend(cfg->backend, params.k, cfg->dense_table_cap));
    if (cfg->max_em_iters < 1) return set_error(PM_ERR_INVALID_PARAMS, "need at least one EM iteration");
    const int64_t r_cap = static_cast<int64_t>(c->t) * params.s;
    if (r_cap > INT32_MAX) return set_error(PM_ERR_UNSUPPORTED, "t*s exceeds 2^31-1");
    PM_CUDA(cudaSetDevice(c->device));
    const int64_t launches0 = c->launches;
    const int64_t h2d0 = c->h2d_bytes, d2h0 = c->d2h_bytes;

    int64_t tb = cfg->trial_begin, te = cfg->trial_end;
    if (tb == 0 && te == 0) {
        tb = 1;
        te = params.m;
    }
    if (tb < 1 || te > params.m || tb > te + 1) return set_error(PM_ERR_INVALID_PARAMS, "trial range must lie within 1..m");
    const int64_t stride = cfg->trial_stride > 1 ? cfg->trial_stride : 1;
    const int64_t n_mine = tb <= te ? (te - tb) / stride + 1 : 0;  // trials tb, tb + stride, ... <= te

    // batch size: bounded by a workspace budget (worst-case per-trial footprint)
    const int key_bytes = 2 * params.k <= 32 ? 4 : 8;
    const int64_t cap_e = std::max<int64_t>(1, c->x / params.s);
    const int64_t tiles = (c->x + k::kSortTile - 1) / k::kSortTile;
    const double per_trial = static_cast<double>(c->x) * (2.0 * key_bytes + 8.0) + 1024.0 * static_cast<double>(tiles) +
                             static_cast<double>(cap_e) * (16.0 + sizeof(k::WorkDesc) + 24.0) + 64.0;
    int64_t batch = cfg->batch_trials > 0 ? cfg->batch_trials
                                          : static_cast<int64_t>(std::max(1.0, std::floor(3.0e9 / per_trial)));
    batch = std::max<int64_t>(1, std::min<int64_t>(batch, 32768));

    RunState st;
    bool stop = false;
    for (int64_t& v : c->em_exact) v = 0;
    HostMarks marks;
    g_marks = &marks;
    struct MarksGuard { ~MarksGuard() { g_marks = nullptr; } } marks_guard;
    host_mark("setup");
    for (int64_t j0 = 0; j0 < n_mine && !stop; j0 += batch) {
        const int64_t first = tb + j0 * stride;  // trial of the batch's first slot
        // Plans come from the reference's PRNG stream (one mt19937_64 per trial, driver.hpp:164):
        // independent per trial, so the host samples them on a few threads.
        const int64_t n_plans = std::min(batch, n_mine - j0);
        std::vector<k::PlanProg> progs(static_cast<size_t>(n_plans));
        std::vector<int> plan_rc(static_cast<size_t>(n_plans), PM_OK);
        // seed-derived plans of a set that takes the one-CTA bucketing are sampled on the device (pm_plans.cuh)
        bool device_plans = cfg->forced_kept == nullptr && cfg->plans == nullptr && fused_hash_applies(c, 2 * params.k, cap_e) &&
                            !(std::getenv("PM_B200_DEVICE_PLANS") != nullptr && std::atoi(std::getenv("PM_B200_DEVICE_PLANS")) == 0);
        auto make_range = [&](int64_t a, int64_t b) {
            if (cfg->forced_kept == nullptr && cfg->plans == nullptr && stride == 1) {
                // the reference's stream, four trials' seed chains at a time (pm_host.cpp: trial_plans)
                std::vector<int32_t> kept(static_cast<size_t>(b - a) * static_cast<size_t>(params.k));
                const int rc = trial_plans(cfg->l, params.k, cfg->seed, first + a, static_cast<int>(b - a), kept.data());
                for (int64_t i = a; i < b; ++i) {
                    plan_rc[static_cast<size_t>(i)] = rc;
                    if (rc == PM_OK) progs[static_cast<size_t>(i)] = make_prog(kept.data() + (i - a) * params.k, params.k);
                }
                return;
            }
            std::vector<int32_t> mine(static_cast<size_t>(params.k));
            for (int64_t i = a; i < b; ++i) {
                const int64_t trial = first + i * stride;
                const int32_t* plan;
                if (cfg->forced_kept != nullptr) {
                    plan = cfg->forced_kept;
                } else if (cfg->plans != nullptr) {
                    plan = cfg->plans + (trial - 1) * params.k;
                    plan_rc[static_cast<size_t>(i)] = validate_plan(cfg->l, plan, params.k);
                } else {
                    plan_rc[static_cast<size_t>(i)] = pm_trial_plan(cfg->l, params.k, cfg->seed, trial, mine.data());
                    plan = mine.data();
                }
                if (plan_rc[static_cast<size_t>(i)] == PM_OK) progs[static_cast<size_t>(i)] = make_prog(plan, params.k);
            }
        };
        const int hw = static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));
        // ~0.3 us per plan (LazyMt64): threads only pay off for thousands of plans
        const int n_threads = static_cast<int>(std::min<int64_t>(std::min(8, hw), (n_plans + 1023) / 1024));
        auto sample_on_host = [&]() {
        if (n_threads <= 1 || cfg->forced_kept != nullptr) {
            make_range(0, n_plans);
        } else {
            std::vector<std::thread> pool;
            const int64_t chunk = (n_plans + n_threads - 1) / n_threads;
            for (int w = 0; w < n_threads; ++w) {
                const int64_t a = w * chunk, b = std::min(n_plans, a + chunk);
                if (a < b) pool.emplace_back(make_range, a, b);
            }
            for (std::thread& th : pool) th.join();
        }
        };
        if (!device_plans) sample_on_host();
        for (int rc_plan : plan_rc) {
            if (rc_plan != PM_OK) return set_error(rc_plan, "invalid projection plan for a trial");
        }
        host_mark("plans");
        auto run_it = [&]() {
            return key_bytes == 4
                       ? run_batch<uint32_t>(c, cfg, params, progs, first, out, &st, &stop, trial_buckets, trial_best_score,
                                             trial_best_expectation, trial_best_key, j0, j0 + n_plans < n_mine || cfg->exact_best != 0, stride, device_plans)
                       : run_batch<uint64_t>(c, cfg, params, progs, first, out, &st, &stop, trial_buckets, trial_best_score,
                                             trial_best_expectation, trial_best_key, j0, j0 + n_plans < n_mine || cfg->exact_best != 0, stride, device_plans);
        };
        int rc = run_it();
        if (rc == kRetryWithHostPlans) {
            device_plans = false;
            sample_on_host();
            for (int rc_plan : plan_rc) {
                if (rc_plan != PM_OK) return set_error(rc_plan, "invalid projection plan for a trial");
            }
            rc = run_it();
        }
        if (rc != PM_OK) return rc;
    }

    out->gpu_launches = c->launches - launches0;
    out->h2d_bytes = c->h2d_bytes - h2d0;
    out->d2h_bytes = c->d2h_bytes - d2h0;
    out->em_fp64_buckets += st.exact_refines;
    out->found = st.have_best ? 1 : 0;
    if (!st.have_best) {
        out->wall_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        return set_error(PM_ERR_NO_ENRICHED_BUCKETS, "no bucket reached s=" + std::to_string(params.s) + " in " +
                                                         std::to_string(out->trials_run) + " trials; lower s or raise m");
    }
    host_mark("reduce+positions");
    if (cfg->exact_best && !st.best_exact && !(st.best_members.empty())) {
        int32_t s64 = 0;
        PM_TRY(exact_candidate(c, cfg, st.best_members, &st.best.expct, &s64));
        st.best_exact = true;
    }
    unpack_consensus(st.best.cons, cfg->l, out->consensus);
    out->score = st.best.score;
    out->iterations = st.best.iters;
    out->expectation = st.best.expct;
    out->source_bucket = st.best.key;
    out->best_trial = st.best_trial;
    if (positions) std::memcpy(positions, st.positions.data(), sizeof(int32_t) * static_cast<size_t>(c->t));
    {
        // XOR/popcount scoring of the reported consensus (north_star "Scoring")
        StageTimer tsc(c, cfg->profile != 0, 5);
        int tot = st.total_distance, within = st.within_d;
        if (!st.ham_valid) PM_TRY(pm_hamming_scan(c, out->consensus, cfg->l, cfg->d, nullptr, &tot, &within));
        out->total_distance = tot;
        out->within_d = within;
    }
    host_mark("hamming");
    collect_stage_times(c, out->stage_ms);
    out->gpu_launches = c->launches - launches0;
    out->h2d_bytes = c->h2d_bytes - h2d0;
    out->d2h_bytes = c->d2h_bytes - d2h0;
    out->wall_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    return PM_OK;
}

// ---- run() on several GPUs of one node ------------------------------------------------------------------
namespace {
struct ShardOut {
    int rc = PM_OK;
    std::string err;
    pm_run_result res{};
    std::vector<int32_t> pos;
    std::vector<int64_t> buckets;  // enriched buckets of each of the shard's trials
    int64_t begin = 0, stride = 1, count = 0;
};
// contexts of pm_run_multi, one per slot of the device list, kept across calls
std::mutex g_multi_mu;
std::vector<pm_ctx*> g_multi_ctx;
}  // namespace

int pm_run_multi(const int* devices, int n_devices, int strided, const pm_run_config* cfg, const char* bases,
                 const int64_t* offs, int t, pm_run_result* out, int32_t* positions) {
    const auto t0 = std::chrono::steady_clock::now();
    clear_error();
    if (devices == nullptr || n_devices < 1 || cfg == nullptr || out == nullptr || bases == nullptr || offs == nullptr) {
        return set_error(PM_ERR_INVALID_PARAMS, "null argument or empty device list");
    }
    std::memset(out, 0, sizeof(*out));
    PM_TRY(pm_resolve_params(cfg, offs, t, out));  // every parameter error surfaces here, before any GPU work
    const pm_run_result params = *out;
    std::lock_guard<std::mutex> lock(g_multi_mu);
    if (static_cast<int>(g_multi_ctx.size()) < n_devices) g_multi_ctx.resize(static_cast<size_t>(n_devices), nullptr);
    for (int i = 0; i < n_devices; ++i) {
        pm_ctx*& c = g_multi_ctx[static_cast<size_t>(i)];
        if (c != nullptr && c->device != devices[i]) {
            pm_ctx_destroy(c);
            c = nullptr;
        }
        if (c == nullptr) PM_TRY(pm_ctx_create(devices[i], nullptr, &c));
    }
    // shards of trials 1..m: contiguous blocks (the remainder spread over the first shards) or round-robin
    const int64_t m = params.m;
    std::vector<ShardOut> parts(static_cast<size_t>(n_devices));
    {
        int64_t next = 1;
        for (int i = 0; i < n_devices; ++i) {
            ShardOut& p = parts[static_cast<size_t>(i)];
            if (strided) {
                p.begin = i + 1;
                p.stride = n_devices;
                p.count = m >= p.begin ? (m - p.begin) / n_devices + 1 : 0;
            } else {
                p.count = m / n_devices + (i < m % n_devices ? 1 : 0);
                p.begin = next;
                p.stride = 1;
                next += p.count;
            }
        }
    }
    auto work = [&](int i) {
        ShardOut& p = parts[static_cast<size_t>(i)];
        if (p.count == 0) return;
        pm_ctx* c = g_multi_ctx[static_cast<size_t>(i)];
        pm_run_config mine = *cfg;
        mine.trial_begin = p.begin;
        mine.trial_end = strided ? m : p.begin + p.count - 1;
        mine.trial_stride = p.stride;
        mine.exact_best = 1;
        p.pos.assign(static_cast<size_t>(t), 0);
        p.buckets.assign(static_cast<size_t>(p.count), 0);
        p.rc = pm_ctx_set_sequences(c, bases, offs, t);
        if (p.rc == PM_OK) p.rc = pm_run(c, &mine, &p.res, p.pos.data(), p.buckets.data(), nullptr, nullptr, nullptr);
        if (p.rc != PM_OK) p.err = pm_last_error();
    };
    {
        std::vector<std::thread> pool;
        for (int i = 1; i < n_devices; ++i) pool.emplace_back(work, i);
        work(0);
        for (std::thread& th : pool) th.join();
    }
    for (const ShardOut& p : parts) {
        if (p.rc != PM_OK && p.rc != PM_ERR_NO_ENRICHED_BUCKETS) return set_error(p.rc, p.err);
    }
    // The ascending-trial scan of driver.hpp:195-208 over the shards: the winner is the maximum under
    // candidate_improves, the earliest trial among exact ties; with early stop the scan ends at the first trial whose
    // candidate is perfect, and only trials up to it count.
    const int perfect = cfg->l * t;
    int64_t stop_trial = m;
    if (cfg->early_stop) {
        for (const ShardOut& p : parts) {
            if (p.res.found && p.res.score == perfect) stop_trial = std::min(stop_trial, p.res.best_trial);
        }
    }
    int winner = -1;
    for (int i = 0; i < n_devices; ++i) {
        const pm_run_result& r = parts[static_cast<size_t>(i)].res;
        if (!r.found || r.best_trial > stop_trial) continue;
        if (winner < 0) {
            winner = i;
            continue;
        }
        const pm_run_result& w = parts[static_cast<size_t>(winner)].res;
        const bool better = pm_candidate_improves(r.score, r.expectation, r.source_bucket, w.score, w.expectation, w.source_bucket) != 0;
        const bool same = r.score == w.score && r.expectation == w.expectation && r.source_bucket == w.source_bucket;
        if (better || (same && r.best_trial < w.best_trial)) winner = i;
    }
    out->trials_run = stop_trial;
    for (const ShardOut& p : parts) {
        for (int64_t j = 0; j < p.count; ++j) {
            if (p.begin + j * p.stride <= stop_trial) out->buckets_enriched += p.buckets[static_cast<size_t>(j)];
        }
        out->gpu_launches += p.res.gpu_launches;
        out->em_lookup_adds += p.res.em_lookup_adds;
        out->em_work += p.res.em_work;
        out->em_tensor_flops += p.res.em_tensor_flops;
        out->em_exact_buckets += p.res.em_exact_buckets;
        out->em_fp64_buckets += p.res.em_fp64_buckets;
        out->h2d_bytes += p.res.h2d_bytes;
        out->d2h_bytes += p.res.d2h_bytes;
        for (int j = 0; j < 8; ++j) out->stage_ms[j] = std::max(out->stage_ms[j], p.res.stage_ms[j]);
    }
    out->wall_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    if (winner < 0) {
        return set_error(PM_ERR_NO_ENRICHED_BUCKETS, "no bucket reached s=" + std::to_string(params.s) + " in " +
                                                         std::to_string(out->trials_run) + " trials; lower s or raise m");
    }
    const ShardOut& w = parts[static_cast<size_t>(winner)];
    std::memcpy(out->consensus, w.res.consensus, sizeof(out->consensus));
    out->score = w.res.score;
    out->iterations = w.res.iterations;
    out->expectation = w.res.expectation;
    out->source_bucket = w.res.source_bucket;
    out->best_trial = w.res.best_trial;
    out->within_d = w.res.within_d;
    out->total_distance = w.res.total_distance;
    out->found = 1;
    if (positions) std::memcpy(positions, w.pos.data(), sizeof(int32_t) * static_cast<size_t>(t));
    return PM_OK;
}

int pm_run_host(pm_ctx* c, const pm_run_config* cfg, const char* bases, const int64_t* offs, int t, pm_run_result* out,
                int32_t* positions) {
    const auto t0 = std::chrono::steady_clock::now();
    if (c == nullptr) return set_error(PM_ERR_INVALID_PARAMS, "null context");
    const int64_t h2d0 = c->h2d_bytes, d2h0 = c->d2h_bytes;
    double up_ms = 0.0;
    {
        const auto a = std::chrono::steady_clock::now();
        PM_TRY(pm_ctx_set_sequences(c, bases, offs, t));
        up_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - a).count();
    }
    const int64_t launches0 = c->launches - 1;
    const int rc = pm_run(c, cfg, out, positions, nullptr, nullptr, nullptr, nullptr);
    out->stage_ms[6] = up_ms;
    out->gpu_launches = c->launches - launches0;
    out->h2d_bytes = c->h2d_bytes - h2d0;
    out->d2h_bytes = c->d2h_bytes - d2h0;
    out->wall_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    return rc;
}

}  // extern "C"
