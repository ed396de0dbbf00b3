// pm_planted.cuh — generate_planted (planted.hpp:38-101) on the device, byte-identical to the reference for the
// same seed.  The reference draws everything from ONE std::mt19937_64 in a contractual order (planted.hpp:30-37):
// the l motif symbols, then per sequence its n background symbols, the start, the d mutated offsets (partial
// Fisher-Yates) and one replacement per offset.  A bounded draw rejects with probability < 1e-16, so the stream has
// a fixed layout: draw q of sequence i sits at  l + i * S + q,  S = n + [W > 1] + 2 d.
//   mt64_stream_kernel   one CTA produces the tempered outputs: the twist of MT19937-64 only reaches 156 words back,
//                        so each half of the 312-word state is 156-way parallel
//   planted_build_kernel one CTA per sequence turns its slice of the stream into ASCII bases, start and mutations
// A rejected draw (which would shift every later draw by one) is detected and reported; the caller then refuses the
// seed (pm_generate_planted on the host handles it) instead of producing different bytes.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace pm {
namespace k {

constexpr int kMtN = 312, kMtM = 156;
constexpr int kMtThreads = 160;

__global__ void __launch_bounds__(kMtThreads) mt64_stream_kernel(uint64_t seed, int64_t n_out, uint64_t* __restrict__ out) {
    __shared__ uint64_t mt[kMtN];
    const int tid = threadIdx.x;
    if (tid == 0) {  // seeding is a dependent chain (one multiply-xor per word)
        uint64_t x = seed;
        mt[0] = x;
        for (int i = 1; i < kMtN; ++i) {
            x = 6364136223846793005ULL * (x ^ (x >> 62)) + static_cast<uint64_t>(i);
            mt[i] = x;
        }
    }
    __syncthreads();
    constexpr uint64_t kUpper = 0xFFFFFFFF80000000ULL, kLower = 0x7FFFFFFFULL, kMatrix = 0xB5026F5AA96619E9ULL;
    for (int64_t base = 0; base < n_out; base += kMtN) {
        // first half: words 0..155 read old words only
        uint64_t v = 0;
        if (tid < kMtM) {
            const uint64_t y = (mt[tid] & kUpper) | (mt[tid + 1] & kLower);
            v = mt[tid + kMtM] ^ (y >> 1) ^ ((y & 1ULL) ? kMatrix : 0ULL);
        }
        __syncthreads();
        if (tid < kMtM) mt[tid] = v;
        __syncthreads();
        // second half: words 156..311 read the new first half (and new word 0 for the last one)
        if (tid < kMtM) {
            const int i = tid + kMtM;
            const uint64_t next = i + 1 < kMtN ? mt[i + 1] : mt[0];
            const uint64_t y = (mt[i] & kUpper) | (next & kLower);
            v = mt[i - kMtM] ^ (y >> 1) ^ ((y & 1ULL) ? kMatrix : 0ULL);
        }
        __syncthreads();
        if (tid < kMtM) mt[tid + kMtM] = v;
        __syncthreads();
        for (int i = tid; i < kMtN; i += kMtThreads) {  // tempering
            if (base + i < n_out) {
                uint64_t x = mt[i];
                x ^= (x >> 29) & 0x5555555555555555ULL;
                x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
                x ^= (x << 37) & 0xFFF7EEE000000000ULL;
                x ^= x >> 43;
                out[base + i] = x;
            }
        }
        __syncthreads();
    }
}

// uniform_below(bound) from one raw output (rng.hpp:37-50); *rejected is raised when the reference would redraw
__device__ __forceinline__ uint64_t planted_below(uint64_t x, uint64_t bound, unsigned int* rejected) {
    if (bound == 1) return 0;
    if (x < (0 - bound) % bound) atomicExch(rejected, 1u);
    return x % bound;
}

__global__ void planted_build_kernel(const uint64_t* __restrict__ draws, int t, int n, int l, int d, char* __restrict__ bases,
                                     char* __restrict__ motif_out, int32_t* __restrict__ positions, unsigned int* __restrict__ rejected) {
    __shared__ int s_start;
    __shared__ int s_off[32];
    __shared__ char s_sym[32];
    const char kSym[4] = {'A', 'C', 'T', 'G'};  // alphabet.hpp:33-36
    const int W = n - l + 1;
    const int64_t per_seq = static_cast<int64_t>(n) + (W > 1 ? 1 : 0) + 2 * d;
    for (int i = blockIdx.x; i < t; i += gridDim.x) {
        const uint64_t* __restrict__ q = draws + l + static_cast<int64_t>(i) * per_seq;
        char* __restrict__ s = bases + static_cast<int64_t>(i) * n;
        __syncthreads();
        if (threadIdx.x == 0) {
            int64_t at = n;
            const int start = W > 1 ? static_cast<int>(planted_below(q[at++], static_cast<uint64_t>(W), rejected)) : 0;
            // d distinct offsets: the first d entries of a partial Fisher-Yates over 1..l (rng.hpp:62-73), then one
            // replacement per offset from the other three symbols (planted.hpp:79-86)
            int pool[32];
            for (int p = 0; p < l; ++p) pool[p] = p + 1;
            for (int m = 0; m < d; ++m) {
                const int j = m + static_cast<int>(planted_below(q[at++], static_cast<uint64_t>(l - m), rejected));
                const int tmp = pool[m];
                pool[m] = pool[j];
                pool[j] = tmp;
            }
            for (int m = 0; m < d; ++m) {
                const int off = pool[m];
                const int old_rank = static_cast<int>(draws[off - 1] & 3ULL);  // the motif's symbol there
                int repl = static_cast<int>(planted_below(q[at++], 3, rejected));
                if (repl >= old_rank) ++repl;
                s_off[m] = off;
                s_sym[m] = kSym[repl];
            }
            s_start = start;
            positions[i] = start + 1;
        }
        __syncthreads();
        const int start = s_start;
        for (int p = threadIdx.x; p < n; p += blockDim.x) {
            char ch = kSym[q[p] & 3ULL];  // uniform_below(4) never rejects: 2^64 mod 4 = 0
            const int c = p - start;
            if (c >= 0 && c < l) {
                ch = kSym[draws[c] & 3ULL];
                for (int m = 0; m < d; ++m) {
                    if (s_off[m] == c + 1) ch = s_sym[m];
                }
            }
            s[p] = ch;
        }
    }
    if (blockIdx.x == 0 && threadIdx.x < l) motif_out[threadIdx.x] = kSym[draws[threadIdx.x] & 3ULL];
}

}  // namespace k
}  // namespace pm
