// pm_plans.cuh — the reference's per-trial projection plans sampled on the device, bit for bit.
//
// Trial i (1-based) seeds its own std::mt19937_64 with splitmix64(master + 0x9E3779B97F4A7C15 (i + 1)) (rng.hpp:13-24,
// driver.hpp:164) and sample_plan (projection.hpp:210-226) draws l - k excluded positions by a partial Fisher-Yates
// over 1..l (rng.hpp:62-73) with the rejection sampler uniform_below (rng.hpp:37-50); the plan is the sorted complement.
// One thread per trial: output o < 156 of MT19937-64 only depends on words o, o + 1 and o + 156 of the seeding chain
// (a dependent multiply-xor recurrence, ~200 steps), so no 312-word state is ever built.  A plan consumes l - k <= 30
// outputs plus rejections (probability < 2^-59 each); a trial that would need more than kPlanMaxOut outputs raises
// *fail and the host samples the batch itself.  The result is the constant-memory extraction program (PlanProg) that
// the hashing kernels read, written to global memory and copied device-to-device into c_plans: the host neither
// samples nor uploads anything (172 plans: 41 us of host arithmetic before the first kernel could start).
#pragma once
#include "pm_kernels.cuh"

namespace pm {
namespace k {

constexpr int kPlanMaxOut = 44;

__device__ __forceinline__ uint64_t plan_splitmix64(uint64_t x) {
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
    return x ^ (x >> 31);
}

__global__ void __launch_bounds__(64) plan_sample_kernel(uint64_t master, int64_t first_trial, int64_t stride, int n, int l, int kk,
                                                       PlanProg* __restrict__ out, int32_t* __restrict__ kept_out /* [n][kk] or null */,
                                                       unsigned int* __restrict__ fail) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint64_t trial = static_cast<uint64_t>(first_trial + static_cast<int64_t>(i) * stride);
    const uint64_t seed = plan_splitmix64(master + 0x9E3779B97F4A7C15ULL * (trial + 1ULL));
    // words 0 .. kPlanMaxOut and 156 .. 156 + kPlanMaxOut - 1 of the seeding chain, in shared memory (one column per
    // thread: dynamically indexed per-thread arrays would live in local memory)
    __shared__ uint64_t s_lo[kPlanMaxOut + 1][64], s_hi[kPlanMaxOut][64];
    const int col = threadIdx.x;
    {
        uint64_t x = seed;
        s_lo[0][col] = x;
        for (int f = 1; f < 156 + kPlanMaxOut; ++f) {
            x = 6364136223846793005ULL * (x ^ (x >> 62)) + static_cast<uint64_t>(f);
            if (f <= kPlanMaxOut) s_lo[f][col] = x;
            if (f >= 156) s_hi[f - 156][col] = x;
        }
    }
    int next = 0;
    bool overflow = false;
    auto draw = [&]() -> uint64_t {
        if (next >= kPlanMaxOut) {
            overflow = true;
            return ~0ULL;
        }
        const int o = next++;
        const uint64_t y = (s_lo[o][col] & (~0ULL << 31)) | (s_lo[o + 1][col] & ((1ULL << 31) - 1ULL));
        uint64_t z = s_hi[o][col] ^ (y >> 1) ^ ((y & 1ULL) ? 0xB5026F5AA96619E9ULL : 0ULL);
        z ^= (z >> 29) & 0x5555555555555555ULL;
        z ^= (z << 17) & 0x71D67FFFEDA60000ULL;
        z ^= (z << 37) & 0xFFF7EEE000000000ULL;
        z ^= z >> 43;
        return z;
    };
    unsigned char pool[32];
    for (int p = 0; p < l; ++p) pool[p] = static_cast<unsigned char>(p + 1);
    const int drop = l - kk;
    for (int a = 0; a < drop; ++a) {
        const uint64_t nn = static_cast<uint64_t>(l - a);
        uint64_t r = 0;
        if (nn != 1) {  // uniform_below(1) consumes nothing
            // nn <= 31: 32-bit arithmetic for the 64-bit remainders (2^32 mod nn, then digit by digit)
            const uint32_t n32 = static_cast<uint32_t>(nn);
            const uint32_t p32 = ((0xFFFFFFFFu % n32) + 1u) % n32;  // 2^32 mod nn
            const uint64_t low_tail = (p32 * p32) % n32;             // 2^64 mod nn = (0 - nn) mod nn
            uint64_t x = draw();
            while (x < low_tail) x = draw();
            r = ((static_cast<uint32_t>(x >> 32) % n32) * p32 + static_cast<uint32_t>(x) % n32) % n32;
        }
        const int b = a + static_cast<int>(r);
        const unsigned char tmp = pool[a];
        pool[a] = pool[b];
        pool[b] = tmp;
    }
    unsigned int dropped = 0;
    for (int a = 0; a < drop; ++a) dropped |= 1u << pool[a];
    if (overflow) atomicExch(fail, 1u);
    // sorted complement -> runs of adjacent kept positions (the host's make_prog)
    PlanProg pp;
    pp.nruns = 0;
    pp.keybits = static_cast<uint8_t>(2 * kk);
    pp.pad[0] = pp.pad[1] = 0;
    for (int r = 0; r < kMaxRuns; ++r) {
        pp.rshift[r] = 0;
        pp.nbits[r] = 0;
    }
    int run = 0, seen = 0;
    for (int p = 1; p <= l + 1; ++p) {
        const bool keep = p <= l && !((dropped >> p) & 1u);
        if (keep) {
            if (kept_out != nullptr) kept_out[static_cast<int64_t>(i) * kk + seen] = p;
            ++seen;
            ++run;
        } else if (run > 0) {
            if (pp.nruns < kMaxRuns) {
                pp.rshift[pp.nruns] = static_cast<uint8_t>(64 - 2 * (p - 1));  // last digit of the run: position p - 1
                pp.nbits[pp.nruns] = static_cast<uint8_t>(2 * run);
                ++pp.nruns;
            }
            run = 0;
        }
    }
    out[i] = pp;
}

}  // namespace k
}  // namespace pm
