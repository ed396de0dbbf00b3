// Restates the reference's own hot-path tests (tests/test_projection.cpp:171-197, :243-249,
// :280-320; tests/test_refine.cpp:154-163; tests/test_driver.cpp:23-38, :86-122, :153-161) against
// the C++ host layer include/projmotif_b200.hpp, which calls the CUDA path through the C ABI.
// Plain asserts (Catch2 is not available); exit code 0 = all passed.
#include <algorithm>
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
    std::printf("host_layer_test: all checks passed\n");
    return 0;
}
