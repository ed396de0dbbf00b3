// Host-only check of the C++ layer's Rng (rng.hpp:25-50): sample_plan must CONSUME the caller's generator, so
// consecutive calls on one Rng give the reference's consecutive plans; next() / uniform_below() / engine() expose the
// same std::mt19937_64 stream.  Prints one line per case; tests/test_host_abi.py compares with the reference goldens.
#include <cstdio>
#include <cstdlib>
#include <random>

#include "projmotif_b200.hpp"

int main(int argc, char** argv) {
    namespace pm = projmotif_b200;
    if (argc < 5) return 2;
    const int l = std::atoi(argv[1]), k = std::atoi(argv[2]), n = std::atoi(argv[4]);
    const std::uint64_t seed = std::strtoull(argv[3], nullptr, 10);
    pm::Rng rng(seed);
    for (int p = 0; p < n; ++p) {
        const pm::ProjectionPlan plan = pm::sample_plan(l, k, rng);
        for (int v : plan.kept_positions()) std::printf("%d ", v);
        std::printf("\n");
    }
    // the generator behind Rng is std::mt19937_64 itself
    pm::Rng a(seed);
    std::mt19937_64 b(seed);
    for (int i = 0; i < 5; ++i) {
        if (a.next() != b()) return 3;
    }
    if (a.engine()() != b()) return 4;
    pm::Rng c(seed);
    std::mt19937_64 d(seed);
    for (std::uint64_t bound : {1ULL, 2ULL, 15ULL, 1000ULL, (1ULL << 63) + 1ULL}) {
        std::uint64_t want = 0;
        if (bound > 1) {
            const std::uint64_t low = (0 - bound) % bound;
            do { want = d(); } while (want < low);
            want %= bound;
        }
        if (c.uniform_below(bound) != want) return 5;
    }
    try {
        c.uniform_below(0);
        return 6;
    } catch (const pm::InvalidParamsError&) {
    }
    std::printf("rng ok\n");
    return 0;
}
