// Restates the reference's own hot-path tests (tests/test_projection.cpp:171-197, :243-249,
// :280-320; tests/test_refine.cpp:154-163; tests/test_driver.cpp:23-38, :86-122, :153-161) against
// the C++ host layer include/projmotif_b200.hpp, which calls the CUDA path through the C ABI.
// Plain asserts (Catch2 is not available); exit code 0 = all passed.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "projmotif_b200.hpp"

using namespace projmotif_b200;

#define REQUIRE(cond)                                                        \
    do {                                                                     \
        if (!(cond)) {                                                       \
            std::fprintf(stderr, "FAILED %s:%d: %s\n", __FILE__, __LINE__, #cond); \
            std::exit(1);                                                    \
        }                                                                    \
    } while (0)

template <typename E, typename F>
static bool throws(F&& f) {
    try {
        f();
    } catch (const E&) {
        return true;
    } catch (...) {
        return false;
    }
    return false;
}

static SequenceSet example_sequences() {
    return SequenceSet({
        "CGGGGCTATGGAACTGGGTCGTCACATTCCCCTTTCGATA", "TTTGAGGGTGCCCAATAAATGCCACTCCAAAGCGGACAAA",
        "GGATGCAACTGATGCCGTTTGACGACCTAAATCAACGGCC", "AAGGATGCAACTCCAGGAGCGCCTTTGCTGGTTCTACCTG",
        "AATTTTCTAAAAAGATTATAATGTCGGTCCATGCAACTTC", "CTGCTGTACAACTGAGATCATGCTGCATGCAACTTTCAAC",
        "TACATGATCTTTTGATGCAACGTGGATGAGGGAATGATGC",
    });
}

int main() {
    const SequenceSet seqs = example_sequences();
    const StartVector starts = {8, 19, 3, 5, 31, 27, 15};
    const std::uint64_t planted_key = 177;  // encode_kmer("ATGAC")

    // hash_trial partitions all l-mers and finds the worked bucket
    const ProjectionPlan plan(8, {1, 2, 3, 6, 7});
    const BucketGrouping grouping = hash_trial(seqs, 8, plan);
    std::size_t total = 0;
    for (std::size_t b = 0; b < grouping.size(); ++b) {
        total += grouping[b].members.size();
        if (b > 0) REQUIRE(grouping[b].key > grouping[b - 1].key);
    }
    REQUIRE(total == seqs.total_lmers(8));
    const auto it = std::find_if(grouping.begin(), grouping.end(), [&](const Bucket& b) { return b.key == planted_key; });
    REQUIRE(it != grouping.end());
    const std::vector<LmerRef> expected = {{1, 8, 8}, {2, 19, 8}, {3, 3, 8}, {4, 5, 8}, {5, 31, 8}, {6, 27, 8}, {7, 15, 8}};
    REQUIRE(it->members == expected);

    // dense backend refuses oversized tables, automatic falls back
    REQUIRE(throws<DenseTableTooLargeError>([&] { hash_trial(seqs, 12, ProjectionPlan::identity(12), HashBackend::dense); }));
    hash_trial(seqs, 12, ProjectionPlan::identity(12), HashBackend::automatic);
    REQUIRE(throws<LengthMismatchError>([&] { hash_trial(seqs, 9, plan); }));
    REQUIRE(throws<InvalidParamsError>([&] { ProjectionPlan(8, {2, 2}); }));

    // enriched_buckets thresholds, sorts and truncates
    const auto enriched = enriched_buckets(seqs, 8, plan, 4, 7 * 4);
    REQUIRE(!enriched.empty());
    REQUIRE(enriched.front().key == planted_key);
    REQUIRE(enriched.front().members.size() == 7);
    REQUIRE(!enriched.front().overflowed);
    const auto capped = enriched_buckets(seqs, 8, plan, 4, 5);
    REQUIRE(capped.front().members.size() == 5 && capped.front().overflowed);
    REQUIRE((capped.front().members.front() == LmerRef{1, 8, 8}));
    REQUIRE(throws<InvalidParamsError>([&] { enriched_buckets(seqs, 8, plan, 0, 5); }));
    REQUIRE(throws<InvalidParamsError>([&] { enriched_buckets(seqs, 8, plan, 3, 2); }));

    // refine converges to the worked consensus
    const RefinedCandidate cand = refine(enriched.front(), seqs, 8);
    REQUIRE(cand.consensus == "ATGCAACT");
    REQUIRE(cand.positions == starts);
    REQUIRE(cand.score == 53);
    REQUIRE(cand.iterations <= 5);
    REQUIRE(cand.expectation > 7.0);
    REQUIRE(cand.source_bucket == planted_key);
    REQUIRE(throws<EmptyBucketError>([&] { refine(EnrichedBucket{}, seqs, 8); }));

    // scoring
    REQUIRE(score(seqs, starts, 8) == 53);
    REQUIRE(consensus(seqs, starts, 8) == "ATGCAACT");
    REQUIRE(total_distance("ATGCAACT", seqs) == 3);

    // resolve_params fills k, s, m from the formulas
    {
        const SequenceSet big(std::vector<std::string>(20, std::string(600, 'A')));
        RunConfig config;
        config.l = 15;
        config.d = 4;
        const TrialParams p = resolve_params(config, big);
        REQUIRE(p.k == 10 && p.s == 3 && p.t_hat == 20);
        REQUIRE(p.m == trials_for_tail(p.q, binomial_lt(p.t_hat, p_hat(15, 4, 10), p.s)));
        RunConfig bad = config;
        bad.l = 5;
        bad.d = 4;
        REQUIRE(throws<InvalidParamsError>([&] { resolve_params(bad, big); }));
        RunConfig unreachable;
        unreachable.l = 8;
        unreachable.d = 6;
        unreachable.k = 1;
        unreachable.s = 1000;
        REQUIRE(throws<UnreachableError>([&] { resolve_params(unreachable, seqs); }));
    }

    // run replays the worked example with a forced plan
    {
        RunConfig config;
        config.l = 8;
        config.d = 1;
        config.s = 4;
        config.forced_kept_positions = std::vector<int>{1, 2, 3, 6, 7};
        const RunResult result = run(config, seqs);
        REQUIRE(result.params.m == 1);
        REQUIRE(result.best.consensus == "ATGCAACT");
        REQUIRE(result.best.score == 53);
        REQUIRE(result.best.positions == starts);
        REQUIRE(result.best.source_bucket == planted_key);
        REQUIRE(result.best_trial == 1 && result.trials_run == 1 && result.buckets_enriched >= 1);
        REQUIRE(result.within_d == 7 && result.total_distance == 3);
    }
    // run reports when no bucket is ever enriched
    {
        RunConfig config;
        config.l = 8;
        config.d = 1;
        config.s = 30;
        config.m = 2;
        REQUIRE(throws<NoEnrichedBucketsError>([&] { run(config, seqs); }));
    }
    REQUIRE(throws<UnknownSymbolError>([] { SequenceSet({"ACGN"}); }));

    // exact solvers (test_oracle.cpp): the median string of the worked example is its motif, and the duality
    // best score = l*t - median distance (test_oracle.cpp:71-80) holds on a toy instance
    {
        const MedianStringResult med = median_string(seqs, 8);
        REQUIRE(med.median == "ATGCAACT" && med.total_distance == 3);
        REQUIRE(throws<SearchSpaceTooLargeError>([&] { median_string(seqs, 8, 1000); }));
        const PlantedInstance toy = generate_planted(3, 12, 4, 1, 17);
        const NaiveMfpResult naive = naive_mfp(toy.sequences, 4);
        const MedianStringResult toy_med = median_string(toy.sequences, 4);
        REQUIRE(naive.score == 4 * 3 - toy_med.total_distance);
        REQUIRE(score(toy.sequences, naive.positions, 4) == naive.score);
        REQUIRE(throws<SearchSpaceTooLargeError>([&] { naive_mfp(toy.sequences, 4, 10); }));
        BenchConfig bench;
        bench.instances = 3;
        bench.run.s = 3;
        const std::string tsv = benchmark(bench);
        REQUIRE(tsv.rfind("instance\tseed\trun_score", 0) == 0);
        REQUIRE(tsv.find("summary\t-\t-\t-\t-\t") != std::string::npos);
    }
    // stage functions of refine.hpp on the device (test_refine.cpp:28-56, :82-127)
    {
        const MotifModel theta0 = init_model(enriched.front().members, seqs, 8, 0.0);
        REQUIRE(theta0.is_column_stochastic());
        // the worked theta0 in sevenths (support.hpp:46-54): the projected columns 1, 2, 3, 6, 7 are unanimous
        // (A, T, G, A, C), the other three hold their consensus symbol six times out of seven
        REQUIRE(std::abs(theta0.at(0, 1) - 1.0) < 1e-12 && std::abs(theta0.at(2, 2) - 1.0) < 1e-12);
        REQUIRE(std::abs(theta0.at(3, 3) - 1.0) < 1e-12 && std::abs(theta0.at(1, 7) - 1.0) < 1e-12);
        REQUIRE(std::abs(theta0.column_max(4) - 6.0 / 7) < 1e-12 && std::abs(theta0.column_max(8) - 6.0 / 7) < 1e-12);
        REQUIRE(std::abs(expectation(theta0) - 53.0 / 7) < 1e-12);
        const MotifModel bg = init_model({{1, 1, 8}}, seqs, 8, 0.0);  // background 76/66/73/65 of 280 (A, C, T, G)
        REQUIRE(std::abs(bg.at(0, 0) - 76.0 / 280) < 1e-12 && std::abs(bg.at(1, 0) - 66.0 / 280) < 1e-12);
        REQUIRE(std::abs(bg.at(2, 0) - 73.0 / 280) < 1e-12 && std::abs(bg.at(3, 0) - 65.0 / 280) < 1e-12);
        REQUIRE(throws<EmptyBucketError>([&] { init_model({}, seqs, 8); }));
        REQUIRE(throws<InvalidParamsError>([&] { init_model({{1, 1, 8}}, seqs, 8, -1.0); }));
        MotifModel uniform(4, 8);
        for (int c = 0; c <= 8; ++c) {
            for (int r = 0; r < 4; ++r) uniform.at(r, c) = 0.25;
        }
        REQUIRE(std::abs(expectation(uniform) - 2.0) < 1e-12);
        REQUIRE(throws<LengthMismatchError>([&] { em_step(uniform, seqs, 7); }));
        // em_step keeps the columns stochastic and never lowers the likelihood (both kernels)
        for (int round = 0; round < 6; ++round) {
            const PlantedInstance inst = generate_planted(5, 30, 6, 1, static_cast<std::uint64_t>(500 + round));
            for (int exact = 0; exact < 2; ++exact) {
                MotifModel model = init_model({{1, inst.positions[0], 6}}, inst.sequences, 6, 0.1);
                double prev = -1e300;
                for (int it = 0; it < 5; ++it) {
                    const EmStepResult step = exact ? em_step_exact(model, inst.sequences, 6) : em_step(model, inst.sequences, 6);
                    REQUIRE(step.model.is_column_stochastic(exact ? 1e-9 : 1e-6));
                    REQUIRE(step.log_likelihood >= prev - (exact ? 1e-6 : 1e-3));
                    prev = step.log_likelihood;
                    model = step.model;
                }
            }
        }
    }
    // run() sharded over a device list (two and three contexts on GPU 0) equals the single-context run,
    // contiguous and round-robin alike
    {
        const PlantedInstance inst = generate_planted(12, 120, 8, 1, 5);
        RunConfig config;
        config.l = 8;
        config.d = 1;
        config.k = 5;
        config.s = 3;
        config.m = 7;
        config.seed = 3;
        config.early_stop = false;
        const RunResult one = run(config, inst.sequences);
        for (int shards = 1; shards <= 3; ++shards) {
            for (int strided = 0; strided < 2; ++strided) {
                RunConfig multi = config;
                multi.devices.assign(static_cast<std::size_t>(shards), 0);
                multi.strided_trials = strided != 0;
                const RunResult r = run(multi, inst.sequences);
                REQUIRE(r.best.consensus == one.best.consensus && r.best.positions == one.best.positions);
                REQUIRE(r.best.score == one.best.score && r.best.source_bucket == one.best.source_bucket);
                REQUIRE(r.best_trial == one.best_trial && r.trials_run == one.trials_run);
                REQUIRE(r.buckets_enriched == one.buckets_enriched);
                REQUIRE(std::abs(r.best.expectation - one.best.expectation) < 1e-4);
            }
        }
    }
    std::printf("host_layer_test: all checks passed\n");
    return 0;
}
