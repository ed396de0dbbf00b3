// ref_shim.cpp — C ABI (oracle/pmo.h) over the UNMODIFIED reference library.
//
// TEST INFRASTRUCTURE ONLY.  This translation unit includes the reference headers where they lie
// (-I/root/reference/proj/include; individual headers, never projmotif.hpp/report.hpp which need
// the un-vendored json.hpp) and forwards every call to the reference's own functions.  It holds
// no algorithm of its own; it exists so that tests and bench.py can run the real reference
// through ctypes.  Built by oracle/Makefile into oracle/_ref/libpm_ref.so (git-ignored).
#include <cstring>
#include <limits>
#include <optional>
#include <string>
#include <vector>

#include <projmotif/driver.hpp>
#include <projmotif/kmer.hpp>
#include <projmotif/oracle.hpp>
#include <projmotif/planted.hpp>
#include <projmotif/projection.hpp>
#include <projmotif/refine.hpp>
#include <projmotif/rng.hpp>
#include <projmotif/scoring.hpp>
#include <projmotif/sequence.hpp>

#include "pmo.h"

using namespace projmotif;

namespace {

thread_local std::string g_error;

int fail(int code, const std::exception& e) {
    g_error = e.what();
    return code;
}

// Maps the reference exception hierarchy (errors.hpp) onto pmo status codes.
template <typename F>
int guarded(F&& f) {
    try {
        g_error.clear();
        f();
        return PMO_OK;
    } catch (const LengthMismatchError& e) {
        return fail(PMO_ERR_LENGTH_MISMATCH, e);
    } catch (const KmerTooLongError& e) {
        return fail(PMO_ERR_KMER_TOO_LONG, e);
    } catch (const DenseTableTooLargeError& e) {
        return fail(PMO_ERR_DENSE_TABLE_TOO_LARGE, e);
    } catch (const SearchSpaceTooLargeError& e) {
        return fail(PMO_ERR_SEARCH_SPACE_TOO_LARGE, e);
    } catch (const UnreachableError& e) {
        return fail(PMO_ERR_UNREACHABLE, e);
    } catch (const EmptyBucketError& e) {
        return fail(PMO_ERR_EMPTY_BUCKET, e);
    } catch (const IndexOutOfRangeError& e) {
        return fail(PMO_ERR_INDEX_OUT_OF_RANGE, e);
    } catch (const InvalidParamsError& e) {
        return fail(PMO_ERR_INVALID_PARAMS, e);
    } catch (const UnknownSymbolError& e) {
        return fail(PMO_ERR_UNKNOWN_SYMBOL, e);
    } catch (const NoEnrichedBucketsError& e) {
        return fail(PMO_ERR_NO_ENRICHED_BUCKETS, e);
    } catch (const NumericalUnderflowError& e) {
        return fail(PMO_ERR_NUMERICAL_UNDERFLOW, e);
    } catch (const std::exception& e) {
        return fail(PMO_ERR_OTHER, e);
    }
}

SequenceSet make_set(const char* bases, const int64_t* offs, int t) {
    std::vector<std::string> seqs;
    seqs.reserve(static_cast<std::size_t>(t));
    for (int i = 0; i < t; ++i) {
        seqs.emplace_back(bases + offs[i], static_cast<std::size_t>(offs[i + 1] - offs[i]));
    }
    return SequenceSet(std::move(seqs), Alphabet::dna());
}

// flat l-mer index (0-based, (seq, offset) order) <-> LmerRef
std::vector<LmerRef> refs_from_flat(const SequenceSet& seqs, int l, const int32_t* flat, int n) {
    std::vector<int64_t> first(static_cast<std::size_t>(seqs.count()) + 1, 0);
    for (int i = 1; i <= seqs.count(); ++i) {
        first[static_cast<std::size_t>(i)] = first[static_cast<std::size_t>(i - 1)] + seqs.window_count(i, l);
    }
    std::vector<LmerRef> out;
    out.reserve(static_cast<std::size_t>(n));
    for (int m = 0; m < n; ++m) {
        int i = 1;
        while (i < seqs.count() && first[static_cast<std::size_t>(i)] <= flat[m]) {
            ++i;
        }
        out.push_back(LmerRef{i, static_cast<int>(flat[m] - first[static_cast<std::size_t>(i - 1)]) + 1, l});
    }
    return out;
}

struct FlatIndexer {
    std::vector<int64_t> first;
    FlatIndexer(const SequenceSet& seqs, int l) : first(static_cast<std::size_t>(seqs.count()) + 1, 0) {
        for (int i = 1; i <= seqs.count(); ++i) {
            first[static_cast<std::size_t>(i)] = first[static_cast<std::size_t>(i - 1)] + seqs.window_count(i, l);
        }
    }
    int32_t operator()(const LmerRef& r) const {
        return static_cast<int32_t>(first[static_cast<std::size_t>(r.seq_index - 1)] + r.offset - 1);
    }
};

RunConfig to_config(const pmo_run_config* c) {
    RunConfig rc;
    rc.l = c->l;
    rc.d = c->d;
    if (c->k != 0) rc.k = c->k;
    if (c->s != 0) rc.s = c->s;
    if (c->m != 0) rc.m = c->m;
    rc.q = c->q;
    rc.seed = c->seed;
    rc.workers = c->workers;
    rc.backend = c->backend == PMO_BACKEND_DENSE     ? HashBackend::dense
                 : c->backend == PMO_BACKEND_GROUPED ? HashBackend::grouped
                                                     : HashBackend::automatic;
    rc.max_em_iters = c->max_em_iters;
    rc.em_tol = c->em_tol;
    rc.s_floor = c->s_floor;
    rc.dense_table_cap = c->dense_table_cap;
    rc.early_stop = c->early_stop != 0;
    if (c->t_hat != 0) rc.t_hat = c->t_hat;
    if (c->forced_kept != nullptr) {
        rc.forced_kept_positions = std::vector<int>(c->forced_kept, c->forced_kept + c->n_forced);
    }
    return rc;
}

void fill_params(const TrialParams& p, pmo_run_result* out) {
    out->k = p.k;
    out->s = p.s;
    out->m = p.m;
    out->q = p.q;
    out->t_hat = p.t_hat;
}

MotifModel model_from(const double* theta, int l) {
    MotifModel m(4, l);
    for (int r = 0; r < 4; ++r) {
        for (int c = 0; c <= l; ++c) {
            m.at(r, c) = theta[r * (l + 1) + c];
        }
    }
    return m;
}

void model_to(const MotifModel& m, int l, double* theta) {
    for (int r = 0; r < 4; ++r) {
        for (int c = 0; c <= l; ++c) {
            theta[r * (l + 1) + c] = m.at(r, c);
        }
    }
}

}  // namespace

extern "C" {

const char* pmo_impl(void) { return "reference"; }
const char* pmo_last_error(void) { return g_error.c_str(); }

void pmo_default_config(pmo_run_config* cfg) {
    const RunConfig d;
    std::memset(cfg, 0, sizeof(*cfg));
    cfg->q = d.q;
    cfg->seed = d.seed;
    cfg->workers = d.workers;
    cfg->backend = PMO_BACKEND_AUTO;
    cfg->max_em_iters = d.max_em_iters;
    cfg->em_tol = d.em_tol;
    cfg->s_floor = d.s_floor;
    cfg->dense_table_cap = d.dense_table_cap;
    cfg->early_stop = d.early_stop ? 1 : 0;
}

uint64_t pmo_splitmix64(uint64_t x) { return splitmix64(x); }
uint64_t pmo_derive_seed(uint64_t master, uint64_t index) { return derive_seed(master, index); }

int pmo_mt_outputs(uint64_t seed, int n, uint64_t* out) {
    return guarded([&] {
        Rng rng(seed);
        for (int i = 0; i < n; ++i) out[i] = rng.next();
    });
}

int pmo_uniform_below(uint64_t seed, uint64_t bound, int n, uint64_t* out) {
    return guarded([&] {
        Rng rng(seed);
        for (int i = 0; i < n; ++i) out[i] = rng.uniform_below(bound);
    });
}

int pmo_sample_plan(int l, int k, uint64_t rng_seed, int32_t* kept) {
    return guarded([&] {
        Rng rng(rng_seed);
        const ProjectionPlan plan = sample_plan(l, k, rng);
        for (int i = 0; i < plan.k(); ++i) kept[i] = plan.kept_positions()[static_cast<std::size_t>(i)];
    });
}

int pmo_sample_plans(int l, int k, uint64_t rng_seed, int n, int32_t* kept) {
    return guarded([&] {
        Rng rng(rng_seed);
        for (int p = 0; p < n; ++p) {
            const ProjectionPlan plan = sample_plan(l, k, rng);
            for (int i = 0; i < plan.k(); ++i) kept[static_cast<std::size_t>(p) * static_cast<std::size_t>(k) + static_cast<std::size_t>(i)] = plan.kept_positions()[static_cast<std::size_t>(i)];
        }
    });
}

int pmo_trial_plan(int l, int k, uint64_t master, int64_t trial, int32_t* kept) {
    return pmo_sample_plan(l, k, derive_seed(master, static_cast<uint64_t>(trial)), kept);
}

int pmo_generate_planted(int t, int n, int l, int d, uint64_t seed, char* bases, char* motif, int32_t* positions) {
    return guarded([&] {
        const PlantedInstance inst = generate_planted(t, n, l, d, seed);
        for (int i = 1; i <= t; ++i) {
            std::memcpy(bases + static_cast<std::size_t>(i - 1) * static_cast<std::size_t>(n),
                        inst.sequences.sequence(i).data(), static_cast<std::size_t>(n));
            positions[i - 1] = inst.positions[static_cast<std::size_t>(i - 1)];
        }
        std::memcpy(motif, inst.motif.data(), static_cast<std::size_t>(l));
    });
}

int pmo_encode_kmer(const char* kmer, int len, uint64_t* out) {
    return guarded([&] { *out = encode_kmer(std::string_view(kmer, static_cast<std::size_t>(len)), Alphabet::dna()); });
}

int pmo_project_encode(const char* lmer, int l, const int32_t* kept, int k, uint64_t* out) {
    return guarded([&] {
        const ProjectionPlan plan(l, std::vector<int>(kept, kept + k));
        *out = project_encode(std::string_view(lmer, static_cast<std::size_t>(l)), plan, Alphabet::dna());
    });
}

int64_t pmo_total_lmers(const int64_t* offs, int t, int l) {
    int64_t x = 0;
    for (int i = 0; i < t; ++i) {
        const int64_t w = (offs[i + 1] - offs[i]) - l + 1;
        if (l < 1 || w < 1) return -1;
        x += w;
    }
    return x;
}

int pmo_hash_keys(const char* bases, const int64_t* offs, int t, int l, const int32_t* kept, int k, uint64_t* keys) {
    return guarded([&] {
        const SequenceSet seqs = make_set(bases, offs, t);
        const ProjectionPlan plan(l, std::vector<int>(kept, kept + k));
        std::size_t i = 0;
        for (const LmerRef& ref : seqs.lmer_refs(l)) {
            keys[i++] = project_encode(seqs.lmer_view(ref), plan, seqs.alphabet());
        }
    });
}

int pmo_hash_trial(const char* bases, const int64_t* offs, int t, int l, const int32_t* kept, int k, int backend,
                   uint64_t dense_cap, int64_t* n_buckets, uint64_t* bucket_keys, int32_t* bucket_sizes,
                   int32_t* members) {
    return guarded([&] {
        const SequenceSet seqs = make_set(bases, offs, t);
        const ProjectionPlan plan(l, std::vector<int>(kept, kept + k));
        const HashBackend hb = backend == PMO_BACKEND_DENSE     ? HashBackend::dense
                               : backend == PMO_BACKEND_GROUPED ? HashBackend::grouped
                                                                : HashBackend::automatic;
        const BucketGrouping grouping = hash_trial(seqs, l, plan, hb, 1, dense_cap);
        const FlatIndexer flat(seqs, l);
        *n_buckets = static_cast<int64_t>(grouping.size());
        std::size_t mpos = 0;
        for (std::size_t b = 0; b < grouping.size(); ++b) {
            bucket_keys[b] = grouping[b].key;
            bucket_sizes[b] = static_cast<int32_t>(grouping[b].members.size());
            for (const LmerRef& r : grouping[b].members) members[mpos++] = flat(r);
        }
    });
}

int pmo_enriched(const char* bases, const int64_t* offs, int t, int l, const int32_t* kept, int k, int s, int r_cap,
                 int64_t* n_enriched, uint64_t* keys, int32_t* sizes_pre, int32_t* overflowed, int64_t* mem_off,
                 int32_t* members) {
    return guarded([&] {
        const SequenceSet seqs = make_set(bases, offs, t);
        const ProjectionPlan plan(l, std::vector<int>(kept, kept + k));
        const BucketGrouping grouping = hash_trial(seqs, l, plan);
        const std::vector<EnrichedBucket> enriched = enriched_buckets(grouping, s, r_cap);
        const FlatIndexer flat(seqs, l);
        *n_enriched = static_cast<int64_t>(enriched.size());
        int64_t mpos = 0;
        for (std::size_t b = 0; b < enriched.size(); ++b) {
            keys[b] = enriched[b].key;
            overflowed[b] = enriched[b].overflowed ? 1 : 0;
            // pre-truncation size: recover it from the grouping
            int32_t pre = static_cast<int32_t>(enriched[b].members.size());
            if (enriched[b].overflowed) {
                for (const Bucket& g : grouping) {
                    if (g.key == enriched[b].key) {
                        pre = static_cast<int32_t>(g.members.size());
                        break;
                    }
                }
            }
            sizes_pre[b] = pre;
            mem_off[b] = mpos;
            for (const LmerRef& r : enriched[b].members) members[mpos++] = flat(r);
        }
        mem_off[enriched.size()] = mpos;
    });
}

int pmo_optimal_k(int l, int d, int* k) {
    return guarded([&] { *k = optimal_k(l, d); });
}
int pmo_p_hat(int l, int d, int k, double* out) {
    return guarded([&] { *out = p_hat(l, d, k); });
}
int pmo_binomial_lt(int t_hat, double p, int s, double* out) {
    return guarded([&] { *out = binomial_lt(t_hat, p, s); });
}
int pmo_trials_for_tail(double q, double miss, int64_t* m) {
    return guarded([&] { *m = trials_for_tail(q, miss); });
}
int pmo_num_trials(double q, int t_hat, double p, int s, int64_t* m) {
    return guarded([&] { *m = num_trials(q, t_hat, p, s); });
}
int pmo_bucket_threshold_for_windows(uint64_t windows, int k, int floor_, int* s) {
    return guarded([&] { *s = bucket_threshold_for_windows(windows, k, floor_); });
}

int pmo_init_model(const char* bases, const int64_t* offs, int t, int l, const int32_t* members, int n_members,
                   double pseudocount, double* theta) {
    return guarded([&] {
        const SequenceSet seqs = make_set(bases, offs, t);
        const MotifModel m = init_model(refs_from_flat(seqs, l, members, n_members), seqs, l, pseudocount);
        model_to(m, l, theta);
    });
}

int pmo_em_step(const char* bases, const int64_t* offs, int t, int l, const double* theta_in, double* theta_out,
                double* log_likelihood) {
    return guarded([&] {
        const SequenceSet seqs = make_set(bases, offs, t);
        const EmStepResult r = em_step(model_from(theta_in, l), seqs, l);
        model_to(r.model, l, theta_out);
        *log_likelihood = r.log_likelihood;
    });
}

int pmo_expectation(const double* theta, int l, double* out) {
    return guarded([&] { *out = expectation(model_from(theta, l)); });
}

int pmo_refine(const char* bases, const int64_t* offs, int t, int l, const int32_t* members, int n_members,
               uint64_t key, int max_iters, double tol, char* consensus, int32_t* positions, int* score,
               double* expectation_out, int* iterations, double* theta_final, double* ll_trace) {
    return guarded([&] {
        const SequenceSet seqs = make_set(bases, offs, t);
        EnrichedBucket bucket;
        bucket.key = key;
        bucket.members = refs_from_flat(seqs, l, members, n_members);
        const RefinedCandidate cand = refine(bucket, seqs, l, max_iters, tol);
        std::memcpy(consensus, cand.consensus.data(), static_cast<std::size_t>(l));
        consensus[l] = '\0';
        for (int i = 0; i < t; ++i) positions[i] = cand.positions[static_cast<std::size_t>(i)];
        *score = cand.score;
        *expectation_out = cand.expectation;
        *iterations = cand.iterations;
        if (theta_final != nullptr || ll_trace != nullptr) {
            // refine() does not expose theta; replay its loop (refine.hpp:293-304) with the
            // reference's own init_model/em_step to obtain the final model and LL trace.
            MotifModel model = init_model(bucket.members, seqs, l, 0.0);
            double prev_ll = -std::numeric_limits<double>::infinity();
            for (int it = 1; it <= max_iters; ++it) {
                EmStepResult step = em_step(model, seqs, l);
                model = std::move(step.model);
                if (ll_trace != nullptr) ll_trace[it - 1] = step.log_likelihood;
                if (it >= 2 && step.log_likelihood - prev_ll < tol) break;
                prev_ll = step.log_likelihood;
            }
            if (theta_final != nullptr) model_to(model, l, theta_final);
        }
    });
}

int pmo_score(const char* bases, const int64_t* offs, int t, int l, const int32_t* starts, int* score_out,
              char* consensus_out) {
    return guarded([&] {
        const SequenceSet seqs = make_set(bases, offs, t);
        const StartVector sv(starts, starts + t);
        *score_out = score(seqs, sv, l);
        const std::string c = consensus(seqs, sv, l);
        std::memcpy(consensus_out, c.data(), static_cast<std::size_t>(l));
        consensus_out[l] = '\0';
    });
}

int pmo_hamming(const char* a, const char* b, int len, int* out) {
    return guarded([&] {
        *out = hamming(std::string_view(a, static_cast<std::size_t>(len)),
                       std::string_view(b, static_cast<std::size_t>(len)));
    });
}

int pmo_total_distance(const char* bases, const int64_t* offs, int t, const char* v, int l, int* total,
                       int32_t* per_seq_min) {
    return guarded([&] {
        const SequenceSet seqs = make_set(bases, offs, t);
        const std::string vv(v, static_cast<std::size_t>(l));
        *total = total_distance(vv, seqs);
        if (per_seq_min != nullptr) {
            for (int i = 1; i <= t; ++i) {
                int best = std::numeric_limits<int>::max();
                for (int j = 1; j <= seqs.window_count(i, l); ++j) {
                    best = std::min(best, hamming(vv, seqs.lmer_view(i, j, l)));
                }
                per_seq_min[i - 1] = best;
            }
        }
    });
}

int pmo_median_string(const char* bases, const int64_t* offs, int t, int l, uint64_t limit, char* median,
                      int* total_distance) {
    return guarded([&] {
        const SequenceSet seqs = make_set(bases, offs, t);
        const MedianStringResult r = median_string(seqs, l, limit);
        std::memcpy(median, r.median.c_str(), r.median.size() + 1);
        *total_distance = r.total_distance;
    });
}

int pmo_naive_mfp(const char* bases, const int64_t* offs, int t, int l, uint64_t limit, int32_t* positions, int* score,
                  char* consensus) {
    return guarded([&] {
        const SequenceSet seqs = make_set(bases, offs, t);
        const NaiveMfpResult r = naive_mfp(seqs, l, limit);
        for (int i = 0; i < t; ++i) positions[i] = r.positions[static_cast<std::size_t>(i)];
        *score = r.score;
        std::memcpy(consensus, r.consensus.c_str(), r.consensus.size() + 1);
    });
}

int pmo_resolve_params(const pmo_run_config* cfg, const char* bases, const int64_t* offs, int t,
                       pmo_run_result* params_out) {
    return guarded([&] {
        const SequenceSet seqs = make_set(bases, offs, t);
        fill_params(resolve_params(to_config(cfg), seqs), params_out);
    });
}

int pmo_run(const pmo_run_config* cfg, const char* bases, const int64_t* offs, int t, pmo_run_result* out,
            int32_t* positions) {
    return guarded([&] {
        const SequenceSet seqs = make_set(bases, offs, t);
        const RunResult r = run(to_config(cfg), seqs);
        std::memset(out, 0, sizeof(*out));
        std::memcpy(out->consensus, r.best.consensus.data(), std::min<std::size_t>(r.best.consensus.size(), 31));
        out->score = r.best.score;
        out->iterations = r.best.iterations;
        out->expectation = r.best.expectation;
        out->source_bucket = r.best.source_bucket;
        out->best_trial = r.best_trial;
        out->trials_run = r.trials_run;
        out->buckets_enriched = r.buckets_enriched;
        out->wall_ms = r.wall_ms;
        fill_params(r.params, out);
        if (positions != nullptr) {
            for (int i = 0; i < t; ++i) positions[i] = r.best.positions[static_cast<std::size_t>(i)];
        }
    });
}

int pmo_trial_outcomes(const pmo_run_config* cfg, const char* bases, const int64_t* offs, int t, int64_t trial_begin,
                       int64_t trial_end, int64_t* buckets, int32_t* best_score, double* best_expectation,
                       uint64_t* best_key) {
    return guarded([&] {
        const SequenceSet seqs = make_set(bases, offs, t);
        const RunConfig config = to_config(cfg);
        const TrialParams params = resolve_params(config, seqs);
        const int r_cap = seqs.count() * params.s;
        std::optional<ProjectionPlan> forced;
        if (config.forced_kept_positions) forced.emplace(config.l, *config.forced_kept_positions);
        // Same calls, same order as run_trial (driver.hpp:163-177).
        for (int64_t trial = trial_begin; trial <= trial_end; ++trial) {
            Rng rng(derive_seed(config.seed, static_cast<uint64_t>(trial)));
            const ProjectionPlan plan = forced ? *forced : sample_plan(params.l, params.k, rng);
            const BucketGrouping grouping =
                hash_trial(seqs, params.l, plan, config.backend, 1, config.dense_table_cap);
            std::optional<RefinedCandidate> best;
            int64_t count = 0;
            for (const EnrichedBucket& bucket : enriched_buckets(grouping, params.s, r_cap)) {
                ++count;
                RefinedCandidate cand = refine(bucket, seqs, params.l, config.max_em_iters, config.em_tol);
                if (!best || detail::candidate_improves(cand, *best)) best = std::move(cand);
            }
            const std::size_t o = static_cast<std::size_t>(trial - trial_begin);
            buckets[o] = count;
            best_score[o] = best ? best->score : -1;
            best_expectation[o] = best ? best->expectation : 0.0;
            best_key[o] = best ? best->source_bucket : 0;
        }
    });
}

}  // extern "C"
