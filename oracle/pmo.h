/*
 * pmo.h — C ABI shared by the two CPU checkers of the PROJECTION hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing under oracle/ is part of the product: only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may load these
 * libraries.  The product (libpm_b200.so) never links or calls them.
 *
 * Two libraries export exactly this interface:
 *   oracle/_ref/libpm_ref.so   — built by oracle/Makefile from oracle/ref_shim.cpp, which #includes
 *                                the UNMODIFIED reference headers in place
 *                                (-I/root/reference/proj/include).  pmo_impl() == "reference".
 *   oracle/libpm_oracle.so     — oracle/pm_oracle.c, a plain-C restatement of the same algorithm
 *                                (each function cites the reference file:line it follows).
 *                                pmo_impl() == "port".
 *
 * Conventions: sequences are passed as one concatenated ASCII buffer `bases` plus `offs[t+1]`
 * (sequence i occupies bases[offs[i] .. offs[i+1])).  "Flat l-mer index" = 0-based rank of an l-mer
 * in the reference's (seq, offset) order (sequence.hpp:122-132).  Positions/starts are 1-based like
 * the reference's public surface.  Every function returns a status code (0 = ok; nonzero mirrors
 * the reference exception type, errors.hpp) and leaves a message in pmo_last_error().
 */
#ifndef PMO_H
#define PMO_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    PMO_OK = 0,
    PMO_ERR_INVALID_PARAMS = 1,        /* errors.hpp:48 InvalidParamsError */
    PMO_ERR_LENGTH_MISMATCH = 2,       /* errors.hpp:44 */
    PMO_ERR_KMER_TOO_LONG = 3,         /* errors.hpp:32 */
    PMO_ERR_DENSE_TABLE_TOO_LARGE = 4, /* errors.hpp:70 */
    PMO_ERR_UNREACHABLE = 5,           /* errors.hpp:76 */
    PMO_ERR_EMPTY_BUCKET = 6,          /* errors.hpp:80 */
    PMO_ERR_NO_ENRICHED_BUCKETS = 7,   /* errors.hpp:85 */
    PMO_ERR_NUMERICAL_UNDERFLOW = 8,   /* errors.hpp:91 */
    PMO_ERR_UNKNOWN_SYMBOL = 9,        /* errors.hpp:28 */
    PMO_ERR_INDEX_OUT_OF_RANGE = 10,   /* errors.hpp:40 */
    PMO_ERR_SEARCH_SPACE_TOO_LARGE = 11, /* errors.hpp:65 */
    PMO_ERR_OTHER = 99
};

enum { PMO_BACKEND_DENSE = 0, PMO_BACKEND_GROUPED = 1, PMO_BACKEND_AUTO = 2 }; /* projection.hpp:91-95 */

/* RunConfig, driver.hpp:23-42.  k, s, m, t_hat: 0 means "not overridden". */
typedef struct pmo_run_config {
    int32_t l, d, k, s;
    int64_t m;
    double q;
    uint64_t seed;
    int32_t workers;
    int32_t backend;
    int32_t max_em_iters;
    int32_t s_floor;
    double em_tol;
    uint64_t dense_table_cap;
    int32_t early_stop;
    int32_t t_hat;
    const int32_t* forced_kept; /* NULL or n_forced 1-based kept positions */
    int32_t n_forced;
    int32_t _pad;
} pmo_run_config;

/* RunResult + TrialParams, driver.hpp:44-52, projection.hpp:23-31. */
typedef struct pmo_run_result {
    char consensus[32]; /* NUL-terminated, l <= 31 */
    int32_t score;
    int32_t iterations;
    double expectation;
    uint64_t source_bucket;
    int64_t best_trial;
    int64_t trials_run;
    int64_t buckets_enriched;
    double wall_ms;
    int32_t k, s;
    int64_t m;
    double q;
    int32_t t_hat;
    int32_t _pad;
} pmo_run_result;

const char* pmo_impl(void);
const char* pmo_last_error(void);
void pmo_default_config(pmo_run_config* cfg); /* RunConfig{} defaults */

/* rng.hpp */
uint64_t pmo_splitmix64(uint64_t x);
uint64_t pmo_derive_seed(uint64_t master, uint64_t index);
int pmo_mt_outputs(uint64_t seed, int n, uint64_t* out);                     /* raw mt19937_64 stream */
int pmo_uniform_below(uint64_t seed, uint64_t bound, int n, uint64_t* out);  /* Rng(seed).uniform_below(bound) x n */
int pmo_sample_plan(int l, int k, uint64_t rng_seed, int32_t* kept);         /* sample_plan(l,k,Rng(rng_seed)) */
int pmo_sample_plans(int l, int k, uint64_t rng_seed, int n, int32_t* kept);     /* n x sample_plan on ONE Rng(rng_seed): kept is n x k */
int pmo_trial_plan(int l, int k, uint64_t master, int64_t trial, int32_t* kept); /* driver.hpp:164-165 */

/* planted.hpp:38-101; bases is t*n chars (no separators), motif l chars, positions t ints */
int pmo_generate_planted(int t, int n, int l, int d, uint64_t seed, char* bases, char* motif, int32_t* positions);

/* kmer.hpp / projection.hpp */
int pmo_encode_kmer(const char* kmer, int len, uint64_t* out);
int pmo_project_encode(const char* lmer, int l, const int32_t* kept, int k, uint64_t* out);
int64_t pmo_total_lmers(const int64_t* offs, int t, int l); /* <0 on error */
int pmo_hash_keys(const char* bases, const int64_t* offs, int t, int l, const int32_t* kept, int k, uint64_t* keys);
int pmo_hash_trial(const char* bases, const int64_t* offs, int t, int l, const int32_t* kept, int k, int backend,
                   uint64_t dense_cap, int64_t* n_buckets, uint64_t* bucket_keys, int32_t* bucket_sizes,
                   int32_t* members /* x flat indices, bucket after bucket */);
int pmo_enriched(const char* bases, const int64_t* offs, int t, int l, const int32_t* kept, int k, int s, int r_cap,
                 int64_t* n_enriched, uint64_t* keys, int32_t* sizes_pre, int32_t* overflowed,
                 int64_t* mem_off /* n_enriched+1 */, int32_t* members /* flat indices */);

/* formulas, projection.hpp:97-206 */
int pmo_optimal_k(int l, int d, int* k);
int pmo_p_hat(int l, int d, int k, double* out);
int pmo_binomial_lt(int t_hat, double p, int s, double* out);
int pmo_trials_for_tail(double q, double miss, int64_t* m);
int pmo_num_trials(double q, int t_hat, double p, int s, int64_t* m);
int pmo_bucket_threshold_for_windows(uint64_t windows, int k, int floor_, int* s);

/* refine.hpp; theta is 4 x (l+1) row-major like MotifModel::index (refine.hpp:65-71) */
int pmo_init_model(const char* bases, const int64_t* offs, int t, int l, const int32_t* members, int n_members,
                   double pseudocount, double* theta);
int pmo_em_step(const char* bases, const int64_t* offs, int t, int l, const double* theta_in, double* theta_out,
                double* log_likelihood);
int pmo_expectation(const double* theta, int l, double* out);
int pmo_refine(const char* bases, const int64_t* offs, int t, int l, const int32_t* members, int n_members,
               uint64_t key, int max_iters, double tol, char* consensus /* l+1 */, int32_t* positions /* t */,
               int* score, double* expectation, int* iterations, double* theta_final /* 4*(l+1) or NULL */,
               double* ll_trace /* max_iters or NULL */);

/* scoring.hpp / oracle.hpp:101-115 */
int pmo_score(const char* bases, const int64_t* offs, int t, int l, const int32_t* starts, int* score,
              char* consensus /* l+1 */);
int pmo_hamming(const char* a, const char* b, int len, int* out);
int pmo_total_distance(const char* bases, const int64_t* offs, int t, const char* v, int l, int* total,
                       int32_t* per_seq_min /* t or NULL */);

/* driver.hpp */
/* exact solvers for small instances, oracle.hpp:45-98 and :120-149 (limits as in the reference: configurations / candidates) */
int pmo_median_string(const char* bases, const int64_t* offs, int t, int l, uint64_t limit, char* median,
                      int* total_distance);
int pmo_naive_mfp(const char* bases, const int64_t* offs, int t, int l, uint64_t limit, int32_t* positions, int* score,
                  char* consensus);

int pmo_resolve_params(const pmo_run_config* cfg, const char* bases, const int64_t* offs, int t, pmo_run_result* params_out);
int pmo_run(const pmo_run_config* cfg, const char* bases, const int64_t* offs, int t, pmo_run_result* out,
            int32_t* positions /* t */);
/* Per-trial view of the same computation as run_trial (driver.hpp:163-177), for trials
 * [trial_begin, trial_end] (1-based, inclusive): enriched-bucket count and the per-trial best. */
int pmo_trial_outcomes(const pmo_run_config* cfg, const char* bases, const int64_t* offs, int t, int64_t trial_begin,
                       int64_t trial_end, int64_t* buckets, int32_t* best_score, double* best_expectation,
                       uint64_t* best_key);

#ifdef __cplusplus
}
#endif
#endif
