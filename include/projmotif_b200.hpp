// projmotif_b200.hpp — C++ host layer over the pm_b200 C ABI with the reference library's own
// entry points, value types and exception types (namespace projmotif -> projmotif_b200), so code
// written against projmotif's hot path compiles against this header by switching the namespace.
//
//   reference (proj/include/projmotif/)                 here
//   errors.hpp            exception hierarchy           same names, thrown from pm_status codes
//   sequence.hpp:19-154   LmerRef, SequenceSet          same (value semantics, 1-based indices)
//   projection.hpp:34-95  ProjectionPlan, Bucket, BucketGrouping, EnrichedBucket, HashBackend
//   projection.hpp:97-206 optimal_k, p_hat, binomial_lt, trials_for_tail, num_trials, bucket_threshold*
//   projection.hpp:210    sample_plan(l, k, Rng&)
//   projection.hpp:319    hash_trial(seqs, l, plan, backend, workers, dense_table_cap)
//   projection.hpp:359    enriched_buckets(grouping, s, r_cap)
//   refine.hpp:288        refine(bucket, seqs, l, max_iters, tol)
//   scoring.hpp:111-131   score, consensus;  sequence.hpp:28 hamming;  oracle.hpp:101 total_distance
//   driver.hpp:23-220     RunConfig, RunResult, TrialParams, resolve_params, run
//
// All heavy work happens in libpm_b200.so on the GPU; nothing here computes the path on the CPU.
// Link with -lpm_b200 (paper_1605_06904_b200/libpm_b200.so).
#pragma once
#include <algorithm>
#include <cctype>
#include <cmath>
#include <charconv>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <initializer_list>
#include <memory>
#include <optional>
#include <stdexcept>
#include <chrono>
#include <random>
#include <string>
#include <string_view>
#include <utility>
#include <vector>

#include "pm_b200.h"

namespace projmotif_b200 {

// ---- errors.hpp
struct Error : std::runtime_error { using std::runtime_error::runtime_error; };
struct ParamError : Error { using Error::Error; };
struct ParseError : Error { using Error::Error; };
struct IoError : Error { using Error::Error; };
struct UnknownSymbolError : ParseError { using ParseError::ParseError; };
struct EmptyInputError : ParseError { using ParseError::ParseError; };
struct RecordWithoutSequenceError : ParseError { using ParseError::ParseError; };
struct FastaFormatError : ParseError { using ParseError::ParseError; };
struct KmerTooLongError : ParamError { using ParamError::ParamError; };
struct IndexOutOfRangeError : ParamError { using ParamError::ParamError; };
struct LengthMismatchError : ParamError { using ParamError::ParamError; };
struct InvalidParamsError : ParamError { using ParamError::ParamError; };
struct DenseTableTooLargeError : ParamError { using ParamError::ParamError; };
struct SearchSpaceTooLargeError : ParamError { using ParamError::ParamError; };
struct UnreachableError : ParamError { using ParamError::ParamError; };
struct EmptyBucketError : ParamError { using ParamError::ParamError; };
struct NoEnrichedBucketsError : Error { using Error::Error; };
struct NumericalUnderflowError : Error { using Error::Error; };
struct DeviceError : Error { using Error::Error; };  // CUDA failure / no B200: there is no CPU fallback

namespace detail {
inline void check(int rc) {
    if (rc == PM_OK) return;
    const std::string msg = pm_last_error();
    switch (rc) {
        case PM_ERR_INVALID_PARAMS: throw InvalidParamsError(msg);
        case PM_ERR_LENGTH_MISMATCH: throw LengthMismatchError(msg);
        case PM_ERR_KMER_TOO_LONG: throw KmerTooLongError(msg);
        case PM_ERR_DENSE_TABLE_TOO_LARGE: throw DenseTableTooLargeError(msg);
        case PM_ERR_UNREACHABLE: throw UnreachableError(msg);
        case PM_ERR_EMPTY_BUCKET: throw EmptyBucketError(msg);
        case PM_ERR_NO_ENRICHED_BUCKETS: throw NoEnrichedBucketsError(msg);
        case PM_ERR_NUMERICAL_UNDERFLOW: throw NumericalUnderflowError(msg);
        case PM_ERR_UNKNOWN_SYMBOL: throw UnknownSymbolError(msg);
        case PM_ERR_INDEX_OUT_OF_RANGE: throw IndexOutOfRangeError(msg);
        case PM_ERR_SEARCH_SPACE_TOO_LARGE: throw SearchSpaceTooLargeError(msg);
        default: throw DeviceError(msg);
    }
}
}  // namespace detail

// ---- sequence.hpp
using StartVector = std::vector<int>;

struct LmerRef {
    int seq_index;
    int offset;
    int length;
    friend bool operator==(const LmerRef& a, const LmerRef& b) {
        return a.seq_index == b.seq_index && a.offset == b.offset && a.length == b.length;
    }
};

class SequenceSet {
public:
    explicit SequenceSet(std::vector<std::string> sequences, std::vector<std::string> names = {})
        : seqs_(std::move(sequences)), names_(std::move(names)) {
        if (seqs_.empty()) throw InvalidParamsError("a sequence set needs at least one sequence");
        if (!names_.empty() && names_.size() != seqs_.size()) {
            throw InvalidParamsError("sequence names must match the sequence count");
        }
        if (names_.empty()) {
            for (std::size_t i = 0; i < seqs_.size(); ++i) names_.push_back("seq" + std::to_string(i + 1));
        }
        offs_.assign(seqs_.size() + 1, 0);
        for (std::size_t i = 0; i < seqs_.size(); ++i) {
            if (seqs_[i].empty()) throw InvalidParamsError("sequence '" + names_[i] + "' is empty");
            for (char c : seqs_[i]) {
                if (c != 'A' && c != 'C' && c != 'G' && c != 'T') {
                    throw UnknownSymbolError(std::string("symbol '") + c + "' in sequence '" + names_[i] +
                                             "' is not in alphabet \"ACTG\"");
                }
            }
            offs_[i + 1] = offs_[i] + static_cast<std::int64_t>(seqs_[i].size());
            bases_ += seqs_[i];
        }
    }
    int count() const { return static_cast<int>(seqs_.size()); }
    int length(int i) const { return static_cast<int>(seqs_.at(static_cast<std::size_t>(i - 1)).size()); }
    const std::string& sequence(int i) const { return seqs_.at(static_cast<std::size_t>(i - 1)); }
    const std::string& name(int i) const { return names_.at(static_cast<std::size_t>(i - 1)); }
    int window_count(int i, int l) const {
        const int w = length(i) - l + 1;
        if (l < 1 || w < 1) throw InvalidParamsError("sequence has no l-mer of length " + std::to_string(l));
        return w;
    }
    std::uint64_t total_lmers(int l) const {
        std::uint64_t x = 0;
        for (int i = 1; i <= count(); ++i) x += static_cast<std::uint64_t>(window_count(i, l));
        return x;
    }
    std::string lmer_at(int i, int j, int l) const {
        const std::string& s = sequence(i);
        if (l < 1 || j < 1 || j + l - 1 > static_cast<int>(s.size())) throw IndexOutOfRangeError("l-mer out of range");
        return s.substr(static_cast<std::size_t>(j - 1), static_cast<std::size_t>(l));
    }
    // C-ABI view
    const std::string& bases() const { return bases_; }
    const std::vector<std::int64_t>& offsets() const { return offs_; }
    // flat l-mer index (0-based, (seq, offset) order) <-> LmerRef
    LmerRef ref_of(std::int64_t flat, int l) const {
        std::int64_t first = 0;
        for (int i = 1; i <= count(); ++i) {
            const std::int64_t w = length(i) - l + 1;
            if (flat < first + w) return LmerRef{i, static_cast<int>(flat - first) + 1, l};
            first += w;
        }
        throw IndexOutOfRangeError("flat l-mer index out of range");
    }
    std::int32_t flat_of(const LmerRef& r) const {
        std::int64_t first = 0;
        for (int i = 1; i < r.seq_index; ++i) first += length(i) - r.length + 1;
        return static_cast<std::int32_t>(first + r.offset - 1);
    }

private:
    std::vector<std::string> seqs_;
    std::vector<std::string> names_;
    std::string bases_;
    std::vector<std::int64_t> offs_;
};

inline int hamming(std::string_view a, std::string_view b) {  // sequence.hpp:28-38 (trivial, host)
    if (a.size() != b.size()) throw LengthMismatchError("hamming distance needs equal lengths");
    int d = 0;
    for (std::size_t i = 0; i < a.size(); ++i) d += a[i] != b[i];
    return d;
}

// ---- device binding: one context per thread, re-uploading only when the SequenceSet changes
class Device {
public:
    static Device& instance() {
        thread_local Device dev;
        return dev;
    }
    pm_ctx* bind(const SequenceSet& seqs) {
        if (!ctx_) {
            pm_ctx* c = nullptr;
            detail::check(pm_ctx_create(device_, nullptr, &c));
            ctx_.reset(c);
        }
        if (loaded_ != seqs.bases() || loaded_offs_ != seqs.offsets()) {
            // a failed upload leaves the context without a set: forget the old one first
            loaded_.clear();
            loaded_offs_.clear();
            detail::check(pm_ctx_set_sequences(ctx_.get(), seqs.bases().data(), seqs.offsets().data(), seqs.count()));
            loaded_ = seqs.bases();
            loaded_offs_ = seqs.offsets();
        }
        return ctx_.get();
    }
    void set_device(int ordinal) {
        ctx_.reset();
        loaded_.clear();
        device_ = ordinal;
    }

private:
    struct Closer {
        void operator()(pm_ctx* c) const { pm_ctx_destroy(c); }
    };
    std::unique_ptr<pm_ctx, Closer> ctx_;
    std::string loaded_;
    std::vector<std::int64_t> loaded_offs_;
    int device_ = 0;
};

// ---- rng.hpp:25-50: std::mt19937_64 (its output for a seed is fixed by the standard) behind a bounded draw that does
// not depend on the standard library's distributions
inline std::uint64_t splitmix64(std::uint64_t x) { return pm_splitmix64(x); }
inline std::uint64_t derive_seed(std::uint64_t master, std::uint64_t index) { return pm_derive_seed(master, index); }
class Rng {
public:
    explicit Rng(std::uint64_t seed) : engine_(seed) {}
    std::uint64_t next() { return engine_(); }
    /// a value in [0, n): outputs below 2^64 mod n are discarded, the rest reduced mod n
    std::uint64_t uniform_below(std::uint64_t n) {
        if (n == 0) throw InvalidParamsError("uniform_below requires a nonempty range");
        if (n == 1) return 0;
        const std::uint64_t discard = (~n + 1) % n;
        for (;;) {
            const std::uint64_t x = engine_();
            if (x >= discard) return x % n;
        }
    }
    std::mt19937_64& engine() { return engine_; }

private:
    std::mt19937_64 engine_;
};

// ---- projection.hpp
struct TrialParams {
    int l = 0, d = 0, k = 0, s = 0;
    std::int64_t m = 0;
    double q = 0.0;
    int t_hat = 0;
};

class ProjectionPlan {
public:
    ProjectionPlan(int l, std::vector<int> kept) : l_(l), kept_(std::move(kept)) {
        detail::check(pm_validate_plan(l_, kept_.data(), static_cast<int>(kept_.size())));
    }
    static ProjectionPlan identity(int l) {
        std::vector<int> all(static_cast<std::size_t>(l));
        for (int p = 1; p <= l; ++p) all[static_cast<std::size_t>(p - 1)] = p;
        return ProjectionPlan(l, std::move(all));
    }
    int l() const { return l_; }
    int k() const { return static_cast<int>(kept_.size()); }
    const std::vector<int>& kept_positions() const { return kept_; }
    bool operator==(const ProjectionPlan& o) const { return l_ == o.l_ && kept_ == o.kept_; }

private:
    int l_;
    std::vector<int> kept_;
};

struct Bucket {
    std::uint64_t key = 0;
    std::vector<LmerRef> members;
};
using BucketGrouping = std::vector<Bucket>;
struct EnrichedBucket {
    std::uint64_t key = 0;
    std::vector<LmerRef> members;
    bool overflowed = false;
};
enum class HashBackend { dense, grouped, automatic };

inline int optimal_k(int l, int d) { int k = 0; detail::check(pm_optimal_k(l, d, &k)); return k; }
inline double p_hat(int l, int d, int k) { double v = 0; detail::check(pm_p_hat(l, d, k, &v)); return v; }
inline double binomial_lt(int t_hat, double p, int s) { double v = 0; detail::check(pm_binomial_lt(t_hat, p, s, &v)); return v; }
inline std::int64_t trials_for_tail(double q, double miss) { std::int64_t m = 0; detail::check(pm_trials_for_tail(q, miss, &m)); return m; }
inline std::int64_t num_trials(double q, int t_hat, double p, int s) { std::int64_t m = 0; detail::check(pm_num_trials(q, t_hat, p, s, &m)); return m; }
inline int bucket_threshold_for_windows(std::uint64_t windows, int k, int floor) {
    int s = 0;
    detail::check(pm_bucket_threshold_for_windows(windows, k, floor, &s));
    return s;
}
inline int bucket_threshold(int t, int n, int l, int k, int floor = 3) {
    if (t < 1 || l < 1 || l > n) throw InvalidParamsError("bucket threshold needs t >= 1 and 1 <= l <= n");
    return bucket_threshold_for_windows(static_cast<std::uint64_t>(t) * static_cast<std::uint64_t>(n - l + 1), k, floor);
}

// sample_plan (projection.hpp:210-226) consumes the caller's generator: two calls on one Rng give two different plans
inline ProjectionPlan sample_plan(int l, int k, Rng& rng) {
    std::vector<int> kept(static_cast<std::size_t>(k > 0 ? k : 1));
    auto pull = [](void* state) -> std::uint64_t { return static_cast<Rng*>(state)->next(); };
    detail::check(pm_sample_plan_stream(l, k, pull, &rng, kept.data()));
    kept.resize(static_cast<std::size_t>(k));
    return ProjectionPlan(l, std::move(kept));
}

inline BucketGrouping hash_trial(const SequenceSet& seqs, int l, const ProjectionPlan& plan,
                                 HashBackend backend = HashBackend::automatic, int /*workers*/ = 1,
                                 std::uint64_t dense_table_cap = 65536) {
    if (plan.l() != l) {
        throw LengthMismatchError("plan built for l=" + std::to_string(plan.l()) + ", asked to hash l=" + std::to_string(l));
    }
    const std::size_t x = static_cast<std::size_t>(seqs.total_lmers(l));
    std::vector<std::uint64_t> keys(x);
    std::vector<std::int32_t> sizes(x), members(x);
    std::int64_t nb = 0;
    const int be = backend == HashBackend::dense ? PM_BACKEND_DENSE : backend == HashBackend::grouped ? PM_BACKEND_GROUPED : PM_BACKEND_AUTO;
    detail::check(pm_hash_trial(Device::instance().bind(seqs), l, plan.kept_positions().data(), plan.k(), be, dense_table_cap,
                                &nb, keys.data(), sizes.data(), members.data()));
    BucketGrouping out(static_cast<std::size_t>(nb));
    std::size_t pos = 0;
    for (std::size_t b = 0; b < out.size(); ++b) {
        out[b].key = keys[b];
        out[b].members.reserve(static_cast<std::size_t>(sizes[b]));
        for (int m = 0; m < sizes[b]; ++m) out[b].members.push_back(seqs.ref_of(members[pos++], l));
    }
    return out;
}

// enriched_buckets (projection.hpp:359-390).  The reference filters a BucketGrouping that hash_trial
// returned by value; its only caller is run_trial (driver.hpp:166-169), which run() below replaces
// wholesale.  Here hashing, threshold, ordering and truncation happen in one device pass, so the
// entry point takes the plan instead of the materialised grouping.
inline std::vector<EnrichedBucket> enriched_buckets(const SequenceSet& seqs, int l, const ProjectionPlan& plan, int s, int r_cap) {
    const std::size_t x = static_cast<std::size_t>(seqs.total_lmers(l));
    std::vector<std::uint64_t> keys(x);
    std::vector<std::int32_t> sizes(x), over(x), members(x);
    std::vector<std::int64_t> moff(x + 1);
    std::int64_t ne = 0;
    detail::check(pm_enriched_buckets(Device::instance().bind(seqs), l, plan.kept_positions().data(), plan.k(), s, r_cap, &ne,
                                      keys.data(), sizes.data(), over.data(), moff.data(), members.data()));
    std::vector<EnrichedBucket> out(static_cast<std::size_t>(ne));
    for (std::size_t b = 0; b < out.size(); ++b) {
        out[b].key = keys[b];
        out[b].overflowed = over[b] != 0;
        for (std::int64_t m = moff[b]; m < moff[b + 1]; ++m) out[b].members.push_back(seqs.ref_of(members[static_cast<std::size_t>(m)], l));
    }
    return out;
}

// ---- refine.hpp
// MotifModel (refine.hpp:20-76): 4 symbol rows x (l+1) columns, column 0 = background; the storage is exactly the
// buffer the C ABI exchanges (row-major, refine.hpp:65-71), so the stage calls below pass data() straight through.
class MotifModel {
public:
    MotifModel(int sigma, int l) : sigma_(sigma), l_(l) {
        if (sigma < 1 || l < 1) throw InvalidParamsError("model dimensions must be positive");
        if (sigma != 4) throw InvalidParamsError("this build models the DNA alphabet only (sigma = 4)");
        cells_.assign(static_cast<std::size_t>(sigma) * static_cast<std::size_t>(l + 1), 0.0);
    }
    int sigma() const { return sigma_; }
    int motif_length() const { return l_; }
    double& at(int rank, int column) { return cells_[slot(rank, column)]; }
    double at(int rank, int column) const { return cells_[slot(rank, column)]; }
    double column_max(int column) const {
        double top = 0.0;
        for (int r = 0; r < sigma_; ++r) top = std::max(top, at(r, column));
        return top;
    }
    bool is_column_stochastic(double tol = 1e-9) const {
        for (int c = 0; c <= l_; ++c) {
            double total = 0.0;
            for (int r = 0; r < sigma_; ++r) {
                const double v = at(r, c);
                if (!(v >= 0.0 && v <= 1.0)) return false;
                total += v;
            }
            if (std::abs(total - 1.0) > tol) return false;
        }
        return true;
    }
    bool operator==(const MotifModel& o) const { return sigma_ == o.sigma_ && l_ == o.l_ && cells_ == o.cells_; }
    double* data() { return cells_.data(); }
    const double* data() const { return cells_.data(); }

private:
    std::size_t slot(int rank, int column) const {
        if (rank < 0 || rank >= sigma_ || column < 0 || column > l_) {
            throw IndexOutOfRangeError("model cell (" + std::to_string(rank) + "," + std::to_string(column) + ") outside " +
                                       std::to_string(sigma_) + "x" + std::to_string(l_ + 1));
        }
        return static_cast<std::size_t>(rank) * static_cast<std::size_t>(l_ + 1) + static_cast<std::size_t>(column);
    }
    int sigma_, l_;
    std::vector<double> cells_;
};

/// init_model (refine.hpp:90-127): theta0 from the members' symbol counts, background from the whole set.
inline MotifModel init_model(const std::vector<LmerRef>& members, const SequenceSet& seqs, int l, double pseudocount = 0.0) {
    if (members.empty()) throw EmptyBucketError("cannot build a motif model from an empty bucket");
    if (pseudocount < 0.0) throw InvalidParamsError("pseudocount must be non-negative");
    std::vector<std::int32_t> flat;
    flat.reserve(members.size());
    for (const LmerRef& r : members) flat.push_back(seqs.flat_of(r));
    MotifModel model(4, l);
    detail::check(pm_init_model(Device::instance().bind(seqs), l, flat.data(), static_cast<int>(flat.size()), pseudocount, model.data()));
    return model;
}

/// expectation (refine.hpp:130-136): sum over the motif columns of the column maximum.
inline double expectation(const MotifModel& model) {
    double e = 0.0;
    detail::check(pm_expectation(model.data(), model.motif_length(), &e));
    return e;
}

struct EmStepResult {
    MotifModel model;
    double log_likelihood = 0.0;  // OOPS log-likelihood of the INPUT model (refine.hpp:209)
};

/// em_step (refine.hpp:216-282) with the production EM kernel; em_step_exact runs the FP64 kernel.
inline EmStepResult em_step(const MotifModel& model, const SequenceSet& seqs, int l) {
    if (model.motif_length() != l) {
        throw LengthMismatchError("model built for l=" + std::to_string(model.motif_length()) + ", asked to step with l=" + std::to_string(l));
    }
    EmStepResult r{MotifModel(4, l), 0.0};
    detail::check(pm_em_step(Device::instance().bind(seqs), l, model.data(), r.model.data(), &r.log_likelihood));
    return r;
}
inline EmStepResult em_step_exact(const MotifModel& model, const SequenceSet& seqs, int l) {
    if (model.motif_length() != l) {
        throw LengthMismatchError("model built for l=" + std::to_string(model.motif_length()) + ", asked to step with l=" + std::to_string(l));
    }
    EmStepResult r{MotifModel(4, l), 0.0};
    detail::check(pm_em_step_exact(Device::instance().bind(seqs), l, model.data(), r.model.data(), &r.log_likelihood));
    return r;
}

struct RefinedCandidate {
    std::string consensus;
    StartVector positions;
    int score = 0;
    double expectation = 0.0;
    int iterations = 0;
    std::uint64_t source_bucket = 0;
};

inline std::vector<RefinedCandidate> refine_all(const std::vector<EnrichedBucket>& buckets, const SequenceSet& seqs, int l,
                                                int max_iters = 5, double tol = 1e-6) {
    if (max_iters < 1) throw InvalidParamsError("need at least one EM iteration");
    const int t = seqs.count();
    std::vector<std::int32_t> members;
    std::vector<std::int64_t> moff(1, 0);
    for (const EnrichedBucket& b : buckets) {
        if (b.members.empty()) throw EmptyBucketError("cannot build a motif model from an empty bucket");
        for (const LmerRef& r : b.members) members.push_back(seqs.flat_of(r));
        moff.push_back(static_cast<std::int64_t>(members.size()));
    }
    const std::size_t nb = buckets.size();
    std::vector<char> cons(32 * (nb ? nb : 1));
    std::vector<std::int32_t> pos(static_cast<std::size_t>(t) * (nb ? nb : 1)), score(nb ? nb : 1), iters(nb ? nb : 1);
    std::vector<double> expct(nb ? nb : 1);
    detail::check(pm_refine(Device::instance().bind(seqs), l, members.data(), moff.data(), static_cast<int>(nb), max_iters, tol,
                            -1.0, cons.data(), pos.data(), score.data(), expct.data(), iters.data(), nullptr, nullptr));
    std::vector<RefinedCandidate> out(nb);
    for (std::size_t b = 0; b < nb; ++b) {
        out[b].consensus.assign(cons.data() + 32 * b, static_cast<std::size_t>(l));
        out[b].positions.assign(pos.begin() + static_cast<std::ptrdiff_t>(b * static_cast<std::size_t>(t)),
                                pos.begin() + static_cast<std::ptrdiff_t>((b + 1) * static_cast<std::size_t>(t)));
        out[b].score = score[b];
        out[b].expectation = expct[b];
        out[b].iterations = iters[b];
        out[b].source_bucket = buckets[b].key;
    }
    return out;
}

inline RefinedCandidate refine(const EnrichedBucket& bucket, const SequenceSet& seqs, int l, int max_iters = 5, double tol = 1e-6) {
    return refine_all({bucket}, seqs, l, max_iters, tol).front();
}

// ---- scoring.hpp / oracle.hpp:101-115
inline int score(const SequenceSet& seqs, const StartVector& starts, int l) {
    if (static_cast<int>(starts.size()) != seqs.count()) throw LengthMismatchError("expected one start per sequence");
    int sc = 0;
    char cons[33];
    detail::check(pm_score(Device::instance().bind(seqs), l, starts.data(), &sc, cons));
    return sc;
}
inline std::string consensus(const SequenceSet& seqs, const StartVector& starts, int l) {
    if (static_cast<int>(starts.size()) != seqs.count()) throw LengthMismatchError("expected one start per sequence");
    int sc = 0;
    char cons[33];
    detail::check(pm_score(Device::instance().bind(seqs), l, starts.data(), &sc, cons));
    return std::string(cons, static_cast<std::size_t>(l));
}
inline int total_distance(const std::string& candidate, const SequenceSet& seqs) {
    int tot = 0;
    detail::check(pm_hamming_scan(Device::instance().bind(seqs), candidate.data(), static_cast<int>(candidate.size()), 0, nullptr, &tot, nullptr));
    return tot;
}

// ---- driver.hpp
struct RunConfig {
    int l = 0;
    int d = 0;
    std::optional<int> k;
    std::optional<int> s;
    std::optional<std::int64_t> m;
    double q = 0.95;
    std::uint64_t seed = 0;
    int workers = 1;
    HashBackend backend = HashBackend::automatic;
    int max_em_iters = 5;
    double em_tol = 1e-6;
    int s_floor = 3;
    std::uint64_t dense_table_cap = 65536;
    bool early_stop = true;
    std::optional<int> t_hat;
    std::optional<std::vector<int>> forced_kept_positions;
    // GPU build: CUDA devices to shard the trials over (empty = the calling thread's device).  The reference
    // parallelises trials over `workers` host threads (driver.hpp:186-209); here the unit is a GPU.  strided_trials
    // deals the trials round-robin instead of in contiguous blocks (results are identical either way).
    std::vector<int> devices;
    bool strided_trials = false;
};

struct RunResult {
    RefinedCandidate best;
    std::int64_t best_trial = 0;
    TrialParams params;
    std::uint64_t seed = 0;
    std::int64_t trials_run = 0;
    std::int64_t buckets_enriched = 0;
    double wall_ms = 0.0;
    // GPU-build extras (north_star "Scoring")
    int within_d = 0;
    int total_distance = 0;
};

namespace detail {
inline pm_run_config to_c(const RunConfig& c) {
    pm_run_config o;
    pm_default_config(&o);
    o.l = c.l;
    o.d = c.d;
    o.k = c.k.value_or(0);
    o.s = c.s.value_or(0);
    o.m = c.m.value_or(0);
    o.q = c.q;
    o.seed = c.seed;
    o.workers = c.workers;
    o.backend = c.backend == HashBackend::dense ? PM_BACKEND_DENSE : c.backend == HashBackend::grouped ? PM_BACKEND_GROUPED : PM_BACKEND_AUTO;
    o.max_em_iters = c.max_em_iters;
    o.em_tol = c.em_tol;
    o.s_floor = c.s_floor;
    o.dense_table_cap = c.dense_table_cap;
    o.early_stop = c.early_stop ? 1 : 0;
    o.t_hat = c.t_hat.value_or(0);
    if (c.forced_kept_positions) {
        o.forced_kept = c.forced_kept_positions->data();
        o.n_forced = static_cast<std::int32_t>(c.forced_kept_positions->size());
    }
    // the reference distinguishes "override = 0/negative" (error) from "no override"; 0 is our
    // "no override" marker, so reject explicit non-positive overrides here like driver.hpp:85-107
    if (c.k && *c.k < 1) throw InvalidParamsError("k override must lie in [1, l]");
    if (c.s && *c.s < 1) throw InvalidParamsError("s override must be at least 1");
    if (c.m && *c.m < 1) throw InvalidParamsError("m override must be at least 1");
    if (c.t_hat && *c.t_hat < 1) throw InvalidParamsError("t_hat must lie in [1, t]");
    return o;
}
}  // namespace detail

inline TrialParams resolve_params(const RunConfig& config, const SequenceSet& seqs) {
    const pm_run_config c = detail::to_c(config);
    pm_run_result r;
    std::memset(&r, 0, sizeof(r));
    detail::check(pm_resolve_params(&c, seqs.offsets().data(), seqs.count(), &r));
    return TrialParams{config.l, config.d, r.k, r.s, r.m, r.q, r.t_hat};
}

inline RunResult run(const RunConfig& config, const SequenceSet& seqs) {
    const pm_run_config c = detail::to_c(config);
    pm_run_result r;
    std::vector<std::int32_t> pos(static_cast<std::size_t>(seqs.count()));
    if (config.devices.empty()) {
        detail::check(pm_run(Device::instance().bind(seqs), &c, &r, pos.data(), nullptr, nullptr, nullptr, nullptr));
    } else {
        detail::check(pm_run_multi(config.devices.data(), static_cast<int>(config.devices.size()), config.strided_trials ? 1 : 0, &c,
                                   seqs.bases().data(), seqs.offsets().data(), seqs.count(), &r, pos.data()));
    }
    RunResult out;
    out.best.consensus = r.consensus;
    out.best.positions.assign(pos.begin(), pos.end());
    out.best.score = r.score;
    out.best.expectation = r.expectation;
    out.best.iterations = r.iterations;
    out.best.source_bucket = r.source_bucket;
    out.best_trial = r.best_trial;
    out.params = TrialParams{config.l, config.d, r.k, r.s, r.m, r.q, r.t_hat};
    out.seed = config.seed;
    out.trials_run = r.trials_run;
    out.buckets_enriched = r.buckets_enriched;
    out.wall_ms = r.wall_ms;
    out.within_d = r.within_d;
    out.total_distance = r.total_distance;
    return out;
}

// ---- FASTA text <-> SequenceSet (behaviour of fasta.hpp:18-97; host text I/O).
// Scanner over the raw bytes: memchr finds the line ends, a record is opened by a line whose FIRST byte is '>',
// residues are folded to upper case with one mask, blanks inside a line are skipped, CR/blank tails are dropped.
namespace detail {
struct FastaRecord {
    std::string name, residues;
};
inline std::string_view drop_tail_blanks(const char* b, const char* e) {
    while (e > b && (e[-1] == '\r' || e[-1] == ' ' || e[-1] == '\t')) --e;
    return std::string_view(b, static_cast<std::size_t>(e - b));
}
inline void require_residues(const std::vector<FastaRecord>& recs) {
    if (!recs.empty() && recs.back().residues.empty()) {
        throw RecordWithoutSequenceError("record '" + recs.back().name + "' has no sequence data");
    }
}
}  // namespace detail

inline SequenceSet parse_fasta(std::string_view text) {
    std::vector<detail::FastaRecord> recs;
    const char* cur = text.data();
    const char* const stop = cur + text.size();
    for (int lineno = 1; cur <= stop; ++lineno) {
        const char* nl = cur < stop ? static_cast<const char*>(std::memchr(cur, '\n', static_cast<std::size_t>(stop - cur))) : nullptr;
        const std::string_view body = detail::drop_tail_blanks(cur, nl ? nl : stop);
        cur = nl ? nl + 1 : stop + 1;
        if (body.empty()) continue;
        if (body[0] == '>') {
            detail::require_residues(recs);
            std::size_t from = 1;
            while (from < body.size() && (body[from] == ' ' || body[from] == '\t')) ++from;
            recs.push_back({std::string(body.substr(from)), std::string()});
            continue;
        }
        if (recs.empty()) throw FastaFormatError("sequence data before the first '>' header at line " + std::to_string(lineno));
        detail::FastaRecord& rec = recs.back();
        for (const char raw : body) {
            if (raw == ' ' || raw == '\t') continue;
            const char up = static_cast<char>(raw & ~0x20);  // 'a'..'z' -> 'A'..'Z'; anything else fails the test below
            if (!(up == 'A' || up == 'C' || up == 'G' || up == 'T') || (raw != up && raw != (up | 0x20))) {
                throw UnknownSymbolError(std::string("unknown symbol '") + raw + "' in record '" + rec.name + "' at line " +
                                         std::to_string(lineno));
            }
            rec.residues.push_back(up);
        }
    }
    if (recs.empty()) throw EmptyInputError("FASTA input contains no records");
    detail::require_residues(recs);
    std::vector<std::string> names, seqs;
    names.reserve(recs.size());
    seqs.reserve(recs.size());
    for (detail::FastaRecord& r : recs) {
        names.push_back(std::move(r.name));
        seqs.push_back(std::move(r.residues));
    }
    return SequenceSet(std::move(seqs), std::move(names));
}

inline std::string serialize_fasta(const SequenceSet& seqs, int line_width = 60) {
    if (line_width < 1) throw InvalidParamsError("FASTA line width must be positive");
    const std::size_t width = static_cast<std::size_t>(line_width);
    std::string text;
    for (int i = 1; i <= seqs.count(); ++i) {
        const std::string& residues = seqs.sequence(i);
        text.reserve(text.size() + seqs.name(i).size() + residues.size() + residues.size() / width + 3);
        text.append(1, '>').append(seqs.name(i)).append(1, '\n');
        for (std::size_t at = 0; at < residues.size(); at += width) text.append(residues, at, width).append(1, '\n');
    }
    return text;
}

// ---- planted.hpp:38-101
struct PlantedInstance {
    SequenceSet sequences;
    std::string motif;
    StartVector positions;
    int l = 0;
    int d = 0;
    std::uint64_t seed = 0;
};

inline PlantedInstance generate_planted(int t, int n, int l, int d, std::uint64_t seed) {
    std::string bases(static_cast<std::size_t>(t > 0 ? t : 0) * static_cast<std::size_t>(n > 0 ? n : 0), 'A');
    std::string motif(static_cast<std::size_t>(l > 0 ? l : 0), 'A');
    std::vector<std::int32_t> pos(static_cast<std::size_t>(t > 0 ? t : 1));
    detail::check(pm_generate_planted(t, n, l, d, seed, bases.data(), motif.data(), pos.data()));
    std::vector<std::string> seqs;
    for (int i = 0; i < t; ++i) seqs.push_back(bases.substr(static_cast<std::size_t>(i) * static_cast<std::size_t>(n), static_cast<std::size_t>(n)));
    return PlantedInstance{SequenceSet(std::move(seqs)), motif, StartVector(pos.begin(), pos.begin() + t), l, d, seed};
}

// ---- report.hpp:15-64 (schema v1).  The reference renders with nlohmann::ordered_json::dump(2);
// the writer below reproduces that layout byte for byte (insertion order, two-space indent, one
// array element per line, shortest round-trip doubles with a trailing ".0" for integral values).
namespace detail {
inline std::string json_double(double v) {
    char buf[64];
    const auto res = std::to_chars(buf, buf + sizeof(buf), v);
    std::string s(buf, res.ptr);
    if (s.find_first_of(".eEn") == std::string::npos) s += ".0";  // 'n' keeps inf/nan untouched
    return s;
}
inline std::string json_string(const std::string& v) {
    std::string out = "\"";
    for (char c : v) {
        switch (c) {
            case '"': out += "\\\""; break;
            case '\\': out += "\\\\"; break;
            case '\n': out += "\\n"; break;
            case '\t': out += "\\t"; break;
            case '\r': out += "\\r"; break;
            default:
                if (static_cast<unsigned char>(c) < 0x20) {
                    char esc[8];
                    std::snprintf(esc, sizeof(esc), "\\u%04x", c);
                    out += esc;
                } else {
                    out += c;
                }
        }
    }
    return out + "\"";
}
inline std::string json_int_array(const std::vector<int>& v, const std::string& indent) {
    if (v.empty()) return "[]";
    std::string out = "[\n";
    for (std::size_t i = 0; i < v.size(); ++i) {
        out += indent + "  " + std::to_string(v[i]) + (i + 1 < v.size() ? ",\n" : "\n");
    }
    return out + indent + "]";
}
inline std::string format_ms(double ms) {  // driver.hpp:237-241
    char buf[32];
    std::snprintf(buf, sizeof(buf), "%.3f", ms);
    return buf;
}
}  // namespace detail

inline constexpr int kResultSchemaVersion = 1;

inline std::string render_result_json(const RunResult& r) {
    std::string o = "{\n";
    o += "  \"version\": " + std::to_string(kResultSchemaVersion) + ",\n";
    o += "  \"params\": {\n";
    o += "    \"l\": " + std::to_string(r.params.l) + ",\n";
    o += "    \"d\": " + std::to_string(r.params.d) + ",\n";
    o += "    \"k\": " + std::to_string(r.params.k) + ",\n";
    o += "    \"s\": " + std::to_string(r.params.s) + ",\n";
    o += "    \"m\": " + std::to_string(r.params.m) + ",\n";
    o += "    \"q\": " + detail::json_double(r.params.q) + ",\n";
    o += "    \"seed\": " + std::to_string(r.seed) + "\n";
    o += "  },\n";
    o += "  \"best\": {\n";
    o += "    \"motif\": " + detail::json_string(r.best.consensus) + ",\n";
    o += "    \"score\": " + std::to_string(r.best.score) + ",\n";
    o += "    \"expectation\": " + detail::json_double(r.best.expectation) + ",\n";
    o += "    \"positions\": " + detail::json_int_array(r.best.positions, "    ") + ",\n";
    o += "    \"source_bucket\": " + std::to_string(r.best.source_bucket) + ",\n";
    o += "    \"trial\": " + std::to_string(r.best_trial) + "\n";
    o += "  },\n";
    o += "  \"stats\": {\n";
    o += "    \"trials_run\": " + std::to_string(r.trials_run) + ",\n";
    o += "    \"buckets_enriched\": " + std::to_string(r.buckets_enriched) + ",\n";
    o += "    \"wall_ms\": " + detail::json_double(r.wall_ms) + "\n";
    o += "  }\n";
    o += "}\n";
    return o;
}

inline std::string render_result_tsv(const RunResult& r) {
    std::string positions;
    for (std::size_t i = 0; i < r.best.positions.size(); ++i) {
        if (i > 0) positions += ',';
        positions += std::to_string(r.best.positions[i]);
    }
    std::string out = "motif\tscore\texpectation\tpositions\tsource_bucket\ttrial\ttrials_run\tbuckets_enriched\twall_ms\n";
    out += r.best.consensus + "\t" + std::to_string(r.best.score) + "\t" + detail::json_double(r.best.expectation) + "\t" +
           positions + "\t" + std::to_string(r.best.source_bucket) + "\t" + std::to_string(r.best_trial) + "\t" +
           std::to_string(r.trials_run) + "\t" + std::to_string(r.buckets_enriched) + "\t" + detail::format_ms(r.wall_ms) + "\n";
    return out;
}

inline std::string truth_json(const PlantedInstance& inst) {
    std::string o = "{\n";
    o += "  \"motif\": " + detail::json_string(inst.motif) + ",\n";
    o += "  \"positions\": " + detail::json_int_array(inst.positions, "  ") + ",\n";
    o += "  \"d\": " + std::to_string(inst.d) + ",\n";
    o += "  \"l\": " + std::to_string(inst.l) + ",\n";
    o += "  \"seed\": " + std::to_string(inst.seed) + "\n";
    o += "}\n";
    return o;
}

// ---- oracle.hpp: exact solvers for small instances
struct NaiveMfpResult {
    StartVector positions;
    int score = 0;
    std::string consensus;
};
struct MedianStringResult {
    std::string median;
    int total_distance = 0;
};

/// median_string (oracle.hpp:120-149) on the device: all 4^l candidates, first minimiser of total_distance in
/// ascending code order (XOR/popcount scan, one thread per candidate).
inline MedianStringResult median_string(const SequenceSet& seqs, int l, std::uint64_t limit = 16777216ULL) {
    MedianStringResult r;
    std::string med(static_cast<std::size_t>(l > 0 ? l : 0) + 1, '\0');
    detail::check(pm_median_string(Device::instance().bind(seqs), l, limit, med.data(), &r.total_distance));
    med.resize(static_cast<std::size_t>(l));
    r.median = med;
    return r;
}

/// naive_mfp (behaviour of oracle.hpp:45-98): the best-scoring start vector over ALL configurations, the first one in
/// lexicographic order (sequence 1 most significant) among equals.  Exponential ground truth for toy instances, plain
/// host C++.  Depth-first over the sequences with one profile per depth; the last sequence is not enumerated through
/// the profile at all: its windows are scored against the column maxima of the prefix in O(l) each.
inline NaiveMfpResult naive_mfp(const SequenceSet& seqs, int l, std::uint64_t limit = 100000000ULL) {
    const int t = seqs.count();
    {   // refuse search spaces beyond the limit (product of the window counts, saturating)
        std::uint64_t configs = 1;
        bool too_many = false;
        for (int i = 1; i <= t && !too_many; ++i) {
            const std::uint64_t w = static_cast<std::uint64_t>(seqs.window_count(i, l));
            too_many = w == 0 || configs > limit / w;
            if (!too_many) configs *= w;
        }
        if (too_many) {
            throw SearchSpaceTooLargeError("naive search needs more than " + std::to_string(limit) +
                                           " configurations; lower t, n, or raise the limit");
        }
    }
    const std::size_t cells = static_cast<std::size_t>(4 * l);
    // 2-bit codes of every sequence (A0 C1 T2 G3, alphabet.hpp:33-36)
    std::vector<std::vector<std::uint8_t>> code(static_cast<std::size_t>(t));
    for (int i = 0; i < t; ++i) {
        const std::string& s = seqs.sequence(i + 1);
        code[static_cast<std::size_t>(i)].resize(s.size());
        for (std::size_t p = 0; p < s.size(); ++p) code[static_cast<std::size_t>(i)][p] = static_cast<std::uint8_t>((static_cast<unsigned char>(s[p]) >> 1) & 3u);
    }
    // depth[i] = profile of the windows chosen for sequences 0..i-1
    std::vector<std::vector<int>> depth(static_cast<std::size_t>(t), std::vector<int>(cells, 0));
    StartVector at(static_cast<std::size_t>(t), 0);  // 0-based start of each sequence on the current path
    NaiveMfpResult best;
    best.score = -1;
    std::vector<int> colmax(static_cast<std::size_t>(l));
    int level = 0;
    at[0] = -1;
    while (level >= 0) {
        const std::size_t lv = static_cast<std::size_t>(level);
        if (level == t - 1) {
            // leaf level: every window of the last sequence against the prefix profile
            const std::vector<int>& pre = depth[lv];
            int base = 0;
            for (int c = 0; c < l; ++c) {
                const int* col = &pre[static_cast<std::size_t>(4 * c)];
                colmax[static_cast<std::size_t>(c)] = std::max(std::max(col[0], col[1]), std::max(col[2], col[3]));
                base += colmax[static_cast<std::size_t>(c)];
            }
            const std::vector<std::uint8_t>& cs = code[lv];
            const int windows = seqs.window_count(t, l);
            for (int j = 0; j < windows; ++j) {
                int sc = base;
                for (int c = 0; c < l; ++c) {
                    // the window's symbol raises its column maximum by one exactly when it already holds the maximum
                    sc += pre[static_cast<std::size_t>(4 * c + cs[static_cast<std::size_t>(j + c)])] == colmax[static_cast<std::size_t>(c)] ? 1 : 0;
                }
                if (sc > best.score) {
                    best.score = sc;
                    best.positions = at;
                    best.positions[lv] = j;
                }
            }
            --level;
            continue;
        }
        // inner level: advance this sequence's start; descend with the extended profile, or backtrack
        if (++at[lv] >= seqs.window_count(level + 1, l)) {
            --level;
            continue;
        }
        std::vector<int>& next = depth[lv + 1];
        next = depth[lv];
        const std::vector<std::uint8_t>& cs = code[lv];
        for (int c = 0; c < l; ++c) ++next[static_cast<std::size_t>(4 * c + cs[static_cast<std::size_t>(at[lv] + c)])];
        ++level;
        if (level < t - 1) at[static_cast<std::size_t>(level)] = -1;
    }
    for (int& p : best.positions) ++p;  // public positions are 1-based
    best.consensus = consensus(seqs, best.positions, l);
    return best;
}

// ---- benchmark() (behaviour of driver.hpp:222-302): the projection pipeline against both exact solvers on planted toy
// instances, one TSV row per instance and a summary row.  BenchConfig mirrors the reference's field names.
struct BenchConfig {
    int instances = 20;
    int t = 3;
    int n = 10;
    int l = 3;
    int d = 1;
    std::uint64_t seed = 1;
    RunConfig run;  // l, d, and seed are overwritten per instance
    std::uint64_t naive_limit = 100000000ULL;
    std::uint64_t median_limit = 16777216ULL;
};

namespace detail {
class Stopwatch {  // wall time of the three solvers, accumulated per column
public:
    template <typename Work>
    double lap(Work&& work) {
        const auto begin = std::chrono::steady_clock::now();
        work();
        const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - begin).count();
        total_ += ms;
        return ms;
    }
    double total() const { return total_; }

private:
    double total_ = 0.0;
};
inline void tsv_row(std::string& out, std::initializer_list<std::string> fields) {
    bool first = true;
    for (const std::string& f : fields) {
        if (!first) out += '\t';
        out += f;
        first = false;
    }
    out += '\n';
}
}  // namespace detail

inline std::string benchmark(const BenchConfig& config) {
    if (config.instances < 1) throw InvalidParamsError("benchmark needs at least one instance");
    std::string report;
    detail::tsv_row(report, {"instance", "seed", "run_score", "oracle_score", "median_distance", "agree", "run_ms", "naive_ms", "median_ms"});
    detail::Stopwatch run_clock, naive_clock, median_clock;
    int agreeing = 0;
    RunConfig per_instance = config.run;
    per_instance.l = config.l;
    per_instance.d = config.d;
    for (int inst_no = 1; inst_no <= config.instances; ++inst_no) {
        per_instance.seed = derive_seed(config.seed, static_cast<std::uint64_t>(inst_no));
        const PlantedInstance inst = generate_planted(config.t, config.n, config.l, config.d, per_instance.seed);
        int found = -1;  // reported when no trial enriches a bucket
        const double run_ms = run_clock.lap([&] {
            try {
                found = run(per_instance, inst.sequences).best.score;
            } catch (const NoEnrichedBucketsError&) {
            }
        });
        NaiveMfpResult exhaustive;
        const double naive_ms = naive_clock.lap([&] { exhaustive = naive_mfp(inst.sequences, config.l, config.naive_limit); });
        MedianStringResult median;
        const double median_ms = median_clock.lap([&] { median = median_string(inst.sequences, config.l, config.median_limit); });
        const bool same = found == exhaustive.score;
        agreeing += same;
        detail::tsv_row(report, {std::to_string(inst_no), std::to_string(per_instance.seed), std::to_string(found),
                                 std::to_string(exhaustive.score), std::to_string(median.total_distance), same ? "true" : "false",
                                 detail::format_ms(run_ms), detail::format_ms(naive_ms), detail::format_ms(median_ms)});
    }
    detail::tsv_row(report, {"summary", "-", "-", "-", "-", std::to_string(agreeing) + "/" + std::to_string(config.instances),
                             detail::format_ms(run_clock.total()), detail::format_ms(naive_clock.total()),
                             detail::format_ms(median_clock.total())});
    return report;
}

}  // namespace projmotif_b200
