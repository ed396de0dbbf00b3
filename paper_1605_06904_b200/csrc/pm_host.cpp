// pm_host.cpp — host-side logic of libpm_b200.so that never touches the GPU:
// status/error plumbing, the projection-plan PRNG stream, the parameter formulas,
// resolve_params and the multi-GPU result merge.  (SURVEY.md §8a rows 3, 13, 14.)
//
// The plan stream must be bit-exact with the reference, so it uses the same standard engine
// (std::mt19937_64, rng.hpp:32) and the same rejection rule (rng.hpp:37-50); plans are sampled on
// the host and shipped to the device as constant-memory extraction programs (paper: "RNG on
// host").
#include <algorithm>
#include <cmath>
#include <cstring>
#include <limits>
#include <memory>
#include <random>
#include <string>
#include <vector>

#include "pm_internal.hpp"

namespace pm {

static thread_local std::string g_last_error;

int set_error(int code, const std::string& msg) {
    g_last_error = msg;
    return code;
}
void clear_error() { g_last_error.clear(); }

uint64_t pow4(int k) {
    if (k >= 32) return std::numeric_limits<uint64_t>::max();
    return 1ULL << (2 * k);
}

int validate_plan(int l, const int32_t* kept, int k) {
    if (l < 1) return set_error(PM_ERR_INVALID_PARAMS, "projection source length must be positive, got " + std::to_string(l));
    if (k < 1 || k > l || kept == nullptr) {
        return set_error(PM_ERR_INVALID_PARAMS, "projection must keep between 1 and l positions, got " +
                                                    std::to_string(k) + " of l=" + std::to_string(l));
    }
    int prev = 0;
    for (int i = 0; i < k; ++i) {
        if (kept[i] <= prev || kept[i] > l) {
            return set_error(PM_ERR_INVALID_PARAMS,
                             "kept positions must be strictly increasing within [1," + std::to_string(l) + "]");
        }
        prev = kept[i];
    }
    return PM_OK;
}

namespace {

// std::mt19937_64 restricted to what a plan needs: the same output stream, produced on demand.  Seeding a
// std::mt19937_64 fills 312 state words and its first output twists all of them (~1 us); a plan consumes
// about l-k outputs, and output i < 156 only depends on seed-chain words i, i+1 and i+156.  The chain is
// extended as far as needed and the words are twisted one at a time; past 156 outputs the standard engine
// takes over (same seed, 156 outputs discarded).  Bit-exactness against std::mt19937_64 is pinned by
// tests/test_host_abi.py.
class LazyMt64 {
public:
    explicit LazyMt64(uint64_t seed) : seed_(seed) { x_[0] = seed; }
    uint64_t operator()() {
        if (next_ >= kM) {
            if (!full_) {
                full_.reset(new std::mt19937_64(seed_));
                full_->discard(kM);
            }
            return (*full_)();
        }
        const int i = next_++;
        extend(i + kM);
        const uint64_t y = (x_[i] & kUpper) | (x_[i + 1] & kLower);
        uint64_t z = x_[i + kM] ^ (y >> 1) ^ ((y & 1ULL) ? 0xB5026F5AA96619E9ULL : 0ULL);
        z ^= (z >> 29) & 0x5555555555555555ULL;
        z ^= (z << 17) & 0x71D67FFFEDA60000ULL;
        z ^= (z << 37) & 0xFFF7EEE000000000ULL;
        z ^= z >> 43;
        return z;
    }

    // advances the seed chains of four engines together up to word `upto` (independent recurrences: ILP)
    static void extend4(LazyMt64& a, LazyMt64& b, LazyMt64& c, LazyMt64& d, int upto) {
        upto = std::min(upto, kN - 1);
        int f = std::max(std::max(a.filled_, b.filled_), std::max(c.filled_, d.filled_));
        a.extend(f), b.extend(f), c.extend(f), d.extend(f);
        for (; f < upto; ++f) {
            const uint64_t pa = a.x_[f], pb = b.x_[f], pc = c.x_[f], pd = d.x_[f];
            const uint64_t add = static_cast<uint64_t>(f + 1);
            a.x_[f + 1] = 6364136223846793005ULL * (pa ^ (pa >> 62)) + add;
            b.x_[f + 1] = 6364136223846793005ULL * (pb ^ (pb >> 62)) + add;
            c.x_[f + 1] = 6364136223846793005ULL * (pc ^ (pc >> 62)) + add;
            d.x_[f + 1] = 6364136223846793005ULL * (pd ^ (pd >> 62)) + add;
        }
        a.filled_ = b.filled_ = c.filled_ = d.filled_ = f;
    }

private:
    static constexpr int kN = 312, kM = 156;
    static constexpr uint64_t kUpper = ~0ULL << 31, kLower = (1ULL << 31) - 1ULL;
    void extend(int upto) {  // seed chain x[i] = f * (x[i-1] ^ (x[i-1] >> 62)) + i
        for (; filled_ < upto; ++filled_) {
            const uint64_t prev = x_[filled_];
            x_[filled_ + 1] = 6364136223846793005ULL * (prev ^ (prev >> 62)) + static_cast<uint64_t>(filled_ + 1);
        }
    }
    uint64_t seed_;
    uint64_t x_[kN];
    int filled_ = 0;  // x_[0..filled_] are valid
    int next_ = 0;
    std::unique_ptr<std::mt19937_64> full_;
};

// Unbiased draw below n by rejecting the low tail 2^64 mod n (rng.hpp:37-50).
template <typename Engine>
uint64_t draw_below(Engine& eng, uint64_t n) {
    if (n == 1) return 0;
    const uint64_t low_tail = (0 - n) % n;
    uint64_t x = eng();
    while (x < low_tail) x = eng();
    return x % n;
}

// sample_plan (projection.hpp:210-226): draw l-k distinct excluded positions by a partial
// Fisher-Yates over 1..l (rng.hpp:62-73); the plan is the sorted complement.
template <typename Engine>
int plan_from_engine(int l, int k, Engine& eng, int32_t* kept) {
    if (k < 1 || k > l) {
        return set_error(PM_ERR_INVALID_PARAMS,
                         "plan needs 1 <= k <= l, got k=" + std::to_string(k) + ", l=" + std::to_string(l));
    }
    constexpr int kStack = 64;  // no heap traffic for the motif lengths of this path
    int pool_s[kStack];
    char dropped_s[kStack + 1];
    std::vector<int> pool_v;
    std::vector<char> dropped_v;
    int* pool = pool_s;
    char* dropped = dropped_s;
    if (l > kStack) {
        pool_v.resize(static_cast<size_t>(l));
        dropped_v.resize(static_cast<size_t>(l) + 1);
        pool = pool_v.data();
        dropped = dropped_v.data();
    }
    for (int i = 0; i < l; ++i) pool[i] = i + 1;
    const int drop = l - k;
    for (int i = 0; i < drop; ++i) {
        const int j = i + static_cast<int>(draw_below(eng, static_cast<uint64_t>(l - i)));
        std::swap(pool[i], pool[j]);
    }
    std::fill(dropped, dropped + l + 1, 0);
    for (int i = 0; i < drop; ++i) dropped[pool[i]] = 1;
    int n = 0;
    for (int p = 1; p <= l; ++p) {
        if (!dropped[p]) kept[n++] = p;
    }
    return PM_OK;
}

}  // namespace

int trial_plans(int l, int k, uint64_t master, int64_t first_trial, int n, int32_t* kept) {
    int i = 0;
    for (; i + 4 <= n; i += 4) {
        LazyMt64 e0(pm_derive_seed(master, static_cast<uint64_t>(first_trial + i))),
            e1(pm_derive_seed(master, static_cast<uint64_t>(first_trial + i + 1))),
            e2(pm_derive_seed(master, static_cast<uint64_t>(first_trial + i + 2))),
            e3(pm_derive_seed(master, static_cast<uint64_t>(first_trial + i + 3)));
        // l - k draws (plus the odd rejection) read words up to 156 + draws; later words are filled on demand
        LazyMt64::extend4(e0, e1, e2, e3, 156 + std::max(0, l - k) + 2);
        LazyMt64* engines[4] = {&e0, &e1, &e2, &e3};
        for (int j = 0; j < 4; ++j) {
            const int rc = plan_from_engine(l, k, *engines[j], kept + static_cast<size_t>(i + j) * static_cast<size_t>(k));
            if (rc != PM_OK) return rc;
        }
    }
    for (; i < n; ++i) {
        const int rc = pm_trial_plan(l, k, master, first_trial + i, kept + static_cast<size_t>(i) * static_cast<size_t>(k));
        if (rc != PM_OK) return rc;
    }
    return PM_OK;
}

namespace {

int64_t total_windows(const int64_t* offs, int t, int l) {
    int64_t x = 0;
    for (int i = 0; i < t; ++i) {
        const int64_t w = (offs[i + 1] - offs[i]) - l + 1;
        if (l < 1 || w < 1) return -1;
        x += w;
    }
    return x;
}

}  // namespace
}  // namespace pm

using namespace pm;

extern "C" {

const char* pm_version(void) { return "pm_b200 0.1 (sm_100a)"; }
const char* pm_last_error(void) { return g_last_error.c_str(); }

void pm_default_config(pm_run_config* cfg) {
    std::memset(cfg, 0, sizeof(*cfg));
    cfg->q = 0.95;
    cfg->workers = 1;
    cfg->backend = PM_BACKEND_AUTO;
    cfg->max_em_iters = 5;
    cfg->em_tol = 1e-6;
    cfg->s_floor = 3;
    cfg->dense_table_cap = 65536;
    cfg->early_stop = 1;
    cfg->z_epsilon = -1.0;
}

uint64_t pm_splitmix64(uint64_t x) {
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
    return x ^ (x >> 31);
}

uint64_t pm_derive_seed(uint64_t master, uint64_t index) {
    return pm_splitmix64(master + 0x9E3779B97F4A7C15ULL * (index + 1));
}

int pm_sample_plan(int l, int k, uint64_t rng_seed, int32_t* kept) {
    clear_error();
    LazyMt64 eng(rng_seed);
    return plan_from_engine(l, k, eng, kept);
}

namespace {
struct CallerStream {  // a generator owned by the caller, pulled one 64-bit output at a time
    uint64_t (*next)(void*);
    void* state;
    uint64_t operator()() { return next(state); }
};
}  // namespace

int pm_sample_plan_stream(int l, int k, uint64_t (*next_u64)(void*), void* state, int32_t* kept) {
    clear_error();
    if (next_u64 == nullptr || kept == nullptr) return set_error(PM_ERR_INVALID_PARAMS, "null argument");
    CallerStream eng{next_u64, state};
    return plan_from_engine(l, k, eng, kept);
}

int pm_trial_plan(int l, int k, uint64_t master, int64_t trial, int32_t* kept) {
    return pm_sample_plan(l, k, pm_derive_seed(master, static_cast<uint64_t>(trial)), kept);
}

int pm_validate_plan(int l, const int32_t* kept, int k) {
    clear_error();
    return validate_plan(l, kept, k);
}

int pm_generate_planted(int t, int n, int l, int d, uint64_t seed, char* bases, char* motif, int32_t* positions) {
    clear_error();
    if (t < 1) return set_error(PM_ERR_INVALID_PARAMS, "need at least one sequence, got t=" + std::to_string(t));
    if (l < 1 || l > n) {
        return set_error(PM_ERR_INVALID_PARAMS, "need 1 <= l <= n, got l=" + std::to_string(l) + ", n=" + std::to_string(n));
    }
    if (d < 0 || d >= l) {
        return set_error(PM_ERR_INVALID_PARAMS, "need 0 <= d < l, got d=" + std::to_string(d) + ", l=" + std::to_string(l));
    }
    static const char kSym[4] = {'A', 'C', 'T', 'G'};
    auto rank_of = [](char c) { return c == 'A' ? 0 : c == 'C' ? 1 : c == 'T' ? 2 : 3; };
    std::mt19937_64 eng(seed);
    // Contractual draw order (planted.hpp:30-37): the motif; then per sequence its n background
    // symbols, the start, the d mutated offsets (partial Fisher-Yates) and one replacement each.
    std::string planted(static_cast<size_t>(l), 'A');
    for (char& c : planted) c = kSym[draw_below(eng, 4)];
    std::vector<int> pool(static_cast<size_t>(l));
    for (int i = 0; i < t; ++i) {
        char* s = bases + static_cast<size_t>(i) * static_cast<size_t>(n);
        for (int p = 0; p < n; ++p) s[p] = kSym[draw_below(eng, 4)];
        const int start = static_cast<int>(draw_below(eng, static_cast<uint64_t>(n - l + 1)));
        std::string occ = planted;
        for (int j = 0; j < l; ++j) pool[static_cast<size_t>(j)] = j;
        for (int j = 0; j < d; ++j) {
            const int pick = j + static_cast<int>(draw_below(eng, static_cast<uint64_t>(l - j)));
            std::swap(pool[static_cast<size_t>(j)], pool[static_cast<size_t>(pick)]);
        }
        for (int j = 0; j < d; ++j) {
            char& c = occ[static_cast<size_t>(pool[static_cast<size_t>(j)])];
            int repl = static_cast<int>(draw_below(eng, 3));
            if (repl >= rank_of(c)) ++repl;  // never redraw the original symbol
            c = kSym[repl];
        }
        std::memcpy(s + start, occ.data(), static_cast<size_t>(l));
        positions[i] = start + 1;
    }
    std::memcpy(motif, planted.data(), static_cast<size_t>(l));
    return PM_OK;
}

int pm_optimal_k(int l, int d, int* k) {
    clear_error();
    if (l - d - 1 < 1) {
        return set_error(PM_ERR_INVALID_PARAMS, "no valid projection width: l-d-1 = " + std::to_string(l - d - 1) +
                                                    " (l=" + std::to_string(l) + ", d=" + std::to_string(d) + ")");
    }
    *k = l - d - 1;
    return PM_OK;
}

int pm_p_hat(int l, int d, int k, double* out) {
    clear_error();
    if (l < 1 || d < 0 || d >= l || k < 0 || k > l) {
        return set_error(PM_ERR_INVALID_PARAMS, "p_hat needs 0 <= d < l and 0 <= k <= l");
    }
    double p = 0.0;
    if (k <= l - d) {
        // C(l-d,k)/C(l,k) as a running product of ratios <= 1, i ascending (same order as the
        // reference so the double result is identical).
        p = 1.0;
        for (int i = 0; i < k; ++i) p *= static_cast<double>(l - d - i) / static_cast<double>(l - i);
    }
    *out = p;
    return PM_OK;
}

int pm_binomial_lt(int t_hat, double p, int s, double* out) {
    clear_error();
    if (t_hat < 1 || s < 0 || p < 0.0 || p > 1.0) {
        return set_error(PM_ERR_INVALID_PARAMS, "binomial_lt needs t_hat >= 1, s >= 0, p in [0,1]");
    }
    double result;
    if (s == 0) {
        result = 0.0;
    } else if (s > t_hat || p <= 0.0) {
        result = 1.0;
    } else if (p >= 1.0) {
        result = 0.0;
    } else {
        // pmf terms built incrementally from (1-p)^t_hat, summed for i = 0 .. s-1
        const double odds = p / (1.0 - p);
        double term = std::pow(1.0 - p, t_hat);
        double acc = term;
        const int last = std::min(s - 1, t_hat);
        for (int i = 0; i < last; ++i) {
            term *= static_cast<double>(t_hat - i) / static_cast<double>(i + 1) * odds;
            acc += term;
        }
        result = std::min(1.0, std::max(0.0, acc));
    }
    *out = result;
    return PM_OK;
}

int pm_trials_for_tail(double q, double miss, int64_t* m_out) {
    clear_error();
    if (!(q > 0.0 && q < 1.0)) return set_error(PM_ERR_INVALID_PARAMS, "q must lie strictly between 0 and 1");
    if (miss >= 1.0) {
        return set_error(PM_ERR_UNREACHABLE, "bucket threshold unattainable: per-trial miss probability is 1");
    }
    if (miss <= 0.0) {
        *m_out = 1;
        return PM_OK;
    }
    // smallest m with miss^m <= 1-q: closed form, then nudged both ways in double arithmetic
    const double target = 1.0 - q;
    const double closed = std::ceil(std::log(target) / std::log(miss));
    int64_t m = closed < 1.0 ? 1 : static_cast<int64_t>(closed);
    while (std::pow(miss, static_cast<double>(m)) > target) ++m;
    while (m > 1 && std::pow(miss, static_cast<double>(m - 1)) <= target) --m;
    *m_out = m;
    return PM_OK;
}

int pm_num_trials(double q, int t_hat, double p, int s, int64_t* m) {
    double miss = 0.0;
    const int rc = pm_binomial_lt(t_hat, p, s, &miss);
    if (rc != PM_OK) return rc;
    return pm_trials_for_tail(q, miss, m);
}

int pm_bucket_threshold_for_windows(uint64_t windows, int k, int floor_, int* s) {
    clear_error();
    if (k < 1 || floor_ < 1) return set_error(PM_ERR_INVALID_PARAMS, "bucket threshold needs k >= 1 and floor >= 1");
    long double buckets = 1.0L;
    for (int i = 0; i < k; ++i) buckets *= 4.0L;
    const long double twice_mean = std::ceil(2.0L * static_cast<long double>(windows) / buckets);
    *s = twice_mean <= static_cast<long double>(floor_) ? floor_ : static_cast<int>(twice_mean);
    return PM_OK;
}

int pm_resolve_params(const pm_run_config* cfg, const int64_t* offs, int t, pm_run_result* params) {
    clear_error();
    if (t < 1) return set_error(PM_ERR_INVALID_PARAMS, "a sequence set needs at least one sequence");
    if (cfg->l < 1) return set_error(PM_ERR_INVALID_PARAMS, "motif length l must be positive");
    if (cfg->d < 0 || cfg->d >= cfg->l) {
        return set_error(PM_ERR_INVALID_PARAMS,
                         "need 0 <= d < l, got d=" + std::to_string(cfg->d) + ", l=" + std::to_string(cfg->l));
    }
    const int64_t windows = total_windows(offs, t, cfg->l);
    if (windows < 0) {
        return set_error(PM_ERR_INVALID_PARAMS, "a sequence has no l-mer of length " + std::to_string(cfg->l));
    }
    params->t_hat = cfg->t_hat != 0 ? cfg->t_hat : t;
    if (params->t_hat < 1 || params->t_hat > t) return set_error(PM_ERR_INVALID_PARAMS, "t_hat must lie in [1, t]");
    if (!(cfg->q > 0.0 && cfg->q < 1.0)) return set_error(PM_ERR_INVALID_PARAMS, "q must lie strictly between 0 and 1");
    params->q = cfg->q;

    int rc;
    if (cfg->forced_kept != nullptr) {
        if ((rc = validate_plan(cfg->l, cfg->forced_kept, cfg->n_forced)) != PM_OK) return rc;
        params->k = cfg->n_forced;
        if (cfg->k != 0 && cfg->k != params->k) {
            return set_error(PM_ERR_INVALID_PARAMS, "k override conflicts with the forced projection plan");
        }
    } else if (cfg->k != 0) {
        if (cfg->k < 1 || cfg->k > cfg->l) return set_error(PM_ERR_INVALID_PARAMS, "k override must lie in [1, l]");
        params->k = cfg->k;
    } else if ((rc = pm_optimal_k(cfg->l, cfg->d, &params->k)) != PM_OK) {
        return rc;
    }

    if (cfg->s != 0) {
        if (cfg->s < 1) return set_error(PM_ERR_INVALID_PARAMS, "s override must be at least 1");
        params->s = cfg->s;
    } else {
        if (cfg->s_floor < 1) return set_error(PM_ERR_INVALID_PARAMS, "s floor must be at least 1");
        rc = pm_bucket_threshold_for_windows(static_cast<uint64_t>(windows), params->k, cfg->s_floor, &params->s);
        if (rc != PM_OK) return rc;
    }

    if (cfg->m != 0) {
        if (cfg->m < 1) return set_error(PM_ERR_INVALID_PARAMS, "m override must be at least 1");
        params->m = cfg->m;
    } else if (cfg->forced_kept != nullptr) {
        params->m = 1;  // a pinned plan makes repeated trials identical (driver.hpp:110-112)
    } else {
        double ph = 0.0;
        if ((rc = pm_p_hat(cfg->l, cfg->d, params->k, &ph)) != PM_OK) return rc;
        rc = pm_num_trials(params->q, params->t_hat, ph, params->s, &params->m);
        if (rc == PM_ERR_UNREACHABLE) {
            return set_error(rc, g_last_error + "; lower s or k, or pass an explicit m");
        }
        if (rc != PM_OK) return rc;
    }
    return PM_OK;
}

int pm_candidate_improves(int score_a, double exp_a, uint64_t key_a, int score_b, double exp_b, uint64_t key_b) {
    if (score_a != score_b) return score_a > score_b;
    if (exp_a != exp_b) return exp_a > exp_b;
    return key_a < key_b;
}

int pm_merge_results(const pm_run_result* parts, const int32_t* const* parts_positions, int n_parts, int t, int l,
                     int early_stop, pm_run_result* out, int32_t* positions_out) {
    clear_error();
    if (n_parts < 1) return set_error(PM_ERR_INVALID_PARAMS, "need at least one partial result");
    // Parts are contiguous trial shards in ascending trial order, so scanning parts in order and
    // replacing only on a strict improvement reproduces the ascending-trial scan of
    // driver.hpp:195-203.  A shard that reached the perfect score ends the scan (driver.hpp:204-207):
    // each shard already truncated itself at its own first perfect trial.
    const int perfect = l * t;
    int winner = -1;
    pm_run_result acc;
    std::memset(&acc, 0, sizeof(acc));
    acc.k = parts[0].k;
    acc.s = parts[0].s;
    acc.m = parts[0].m;
    acc.q = parts[0].q;
    acc.t_hat = parts[0].t_hat;
    for (int i = 0; i < n_parts; ++i) {
        const pm_run_result& p = parts[i];
        acc.trials_run = std::max(acc.trials_run, p.trials_run);
        acc.buckets_enriched += p.buckets_enriched;
        acc.wall_ms = std::max(acc.wall_ms, p.wall_ms);
        acc.gpu_launches += p.gpu_launches;
        acc.em_lookup_adds += p.em_lookup_adds;
        acc.em_work += p.em_work;
        acc.em_tensor_flops += p.em_tensor_flops;
        acc.em_exact_buckets += p.em_exact_buckets;
        acc.em_fp64_buckets += p.em_fp64_buckets;
        acc.h2d_bytes += p.h2d_bytes;
        acc.d2h_bytes += p.d2h_bytes;
        for (int j = 0; j < 8; ++j) acc.stage_ms[j] = std::max(acc.stage_ms[j], p.stage_ms[j]);
        if (p.found && (winner < 0 || pm_candidate_improves(p.score, p.expectation, p.source_bucket, acc.score,
                                                            acc.expectation, acc.source_bucket))) {
            winner = i;
            std::memcpy(acc.consensus, p.consensus, sizeof(acc.consensus));
            acc.score = p.score;
            acc.iterations = p.iterations;
            acc.expectation = p.expectation;
            acc.source_bucket = p.source_bucket;
            acc.best_trial = p.best_trial;
            acc.within_d = p.within_d;
            acc.total_distance = p.total_distance;
            acc.found = 1;
        }
        if (early_stop && acc.found && acc.score == perfect) {
            acc.trials_run = p.trials_run;
            break;
        }
    }
    *out = acc;
    if (winner < 0) {
        return set_error(PM_ERR_NO_ENRICHED_BUCKETS, "no bucket reached s=" + std::to_string(acc.s) + " in " +
                                                         std::to_string(acc.trials_run) +
                                                         " trials; lower s or raise m");
    }
    if (positions_out != nullptr && parts_positions != nullptr && parts_positions[winner] != nullptr) {
        std::memcpy(positions_out, parts_positions[winner], sizeof(int32_t) * static_cast<size_t>(t));
    }
    return PM_OK;
}

}  // extern "C"
