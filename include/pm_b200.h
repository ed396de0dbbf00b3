/*
 * pm_b200.h — C ABI of libpm_b200.so, the B200 (sm_100a) implementation of the PROJECTION
 * motif-finding hot path of the `projmotif` reference library (arXiv 1605.06904).
 *
 * This is the drop-in boundary.  The reference has no FFI or plugin registry: the path sits
 * behind inline C++ functions in namespace projmotif.  Each entry point below
 * names the reference function it replaces (file:line under /root/reference/proj/include/
 * projmotif/); include/projmotif_b200.hpp is the C++ host layer that gives these the
 * reference's own signatures, value types and exception types.
 *
 * Conventions
 *  - plain pointers and sizes; no STL, no exceptions, no torch types cross this boundary;
 *  - sequences: one concatenated ASCII buffer `bases` (upper-case A,C,G,T) + `offs[t+1]`, sequence
 *    i = bases[offs[i] .. offs[i+1]);
 *  - public positions are 1-based like the reference; "flat l-mer index" is the 0-based rank of
 *    an l-mer in the reference's (seq, offset) order (sequence.hpp:122-132);
 *  - every function returns a pm_status (0 = ok).  Nonzero codes 1..10 mirror the reference
 *    exception types (errors.hpp); pm_last_error() returns the thread-local message;
 *  - symbol code A0 C1 T2 G3 (alphabet.hpp:33-36); keys are base-4 Horner codes with the first
 *    kept position as the most significant digit (projection.hpp:243-254);
 *  - there is NO CPU fallback: device entry points fail with PM_ERR_NO_DEVICE / PM_ERR_CUDA when
 *    no sm_100 GPU is usable.  Host-only entry points (section 1) never touch the GPU.
 */
#ifndef PM_B200_H
#define PM_B200_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum pm_status {
    PM_OK = 0,
    PM_ERR_INVALID_PARAMS = 1,        /* errors.hpp:48 InvalidParamsError */
    PM_ERR_LENGTH_MISMATCH = 2,       /* errors.hpp:44 LengthMismatchError */
    PM_ERR_KMER_TOO_LONG = 3,         /* errors.hpp:32 KmerTooLongError */
    PM_ERR_DENSE_TABLE_TOO_LARGE = 4, /* errors.hpp:70 DenseTableTooLargeError */
    PM_ERR_UNREACHABLE = 5,           /* errors.hpp:76 UnreachableError */
    PM_ERR_EMPTY_BUCKET = 6,          /* errors.hpp:80 EmptyBucketError */
    PM_ERR_NO_ENRICHED_BUCKETS = 7,   /* errors.hpp:85 NoEnrichedBucketsError */
    PM_ERR_NUMERICAL_UNDERFLOW = 8,   /* errors.hpp:91 NumericalUnderflowError */
    PM_ERR_UNKNOWN_SYMBOL = 9,        /* errors.hpp:28 UnknownSymbolError */
    PM_ERR_INDEX_OUT_OF_RANGE = 10,   /* errors.hpp:40 IndexOutOfRangeError */
    PM_ERR_SEARCH_SPACE_TOO_LARGE = 11, /* errors.hpp:65 SearchSpaceTooLargeError */
    PM_ERR_UNSUPPORTED = 50,          /* valid for the reference, outside this build's limits (e.g. l > 31) */
    PM_ERR_CUDA = 100,                /* a CUDA runtime call or kernel failed */
    PM_ERR_NO_DEVICE = 101,           /* no usable sm_100 device: there is no CPU fallback */
    PM_ERR_OUT_OF_MEMORY = 102
} pm_status;

enum { PM_BACKEND_DENSE = 0, PM_BACKEND_GROUPED = 1, PM_BACKEND_AUTO = 2 }; /* projection.hpp:91-95 */
#define PM_MAX_L 31 /* any l-mer fits one 64-bit word at 2 bits/base */

/* RunConfig (driver.hpp:23-42) followed by the fields that only exist on the GPU build.
 * k, s, m, t_hat: 0 = not overridden (reference: std::nullopt). */
typedef struct pm_run_config {
    int32_t l, d, k, s;
    int64_t m;
    double q;
    uint64_t seed;
    int32_t workers;          /* accepted, no effect on results (driver.hpp:148) */
    int32_t backend;          /* PM_BACKEND_*: validated like projection.hpp:341-351; results identical */
    int32_t max_em_iters;
    int32_t s_floor;
    double em_tol;
    uint64_t dense_table_cap;
    int32_t early_stop;
    int32_t t_hat;
    const int32_t* forced_kept; /* forced_kept_positions (driver.hpp:39-41): NULL or n_forced 1-based positions */
    int32_t n_forced;
    int32_t _pad0;
    /* ---- extensions (all default to 0 = reference behaviour) ---- */
    const int32_t* plans;     /* optional explicit m x k kept positions (1-based), one plan per trial */
    int64_t trial_begin;      /* multi-GPU sharding: run trials [trial_begin, trial_end] of 1..m; 0,0 = all */
    int64_t trial_end;
    int32_t batch_trials;     /* trials per device batch; 0 = auto */
    int32_t profile;          /* 1: time each stage with CUDA events into pm_run_result.stage_ms */
    double z_epsilon;         /* M-step responsibility cut-off; <0 = default (2^-30); 0 = every window */
    int64_t trial_stride;     /* 0/1: every trial of [trial_begin, trial_end]; N > 1: trial_begin, trial_begin+N, ... (round-robin
                                 shards: the right split when the answer is expected within the first few trials) */
    int32_t exact_best;       /* 1: the reported winner's expectation is the FP64 kernel's (what a cross-shard comparison of
                                 near-equal candidates needs) */
    int32_t _pad1;
} pm_run_config;

/* RunResult + TrialParams (driver.hpp:44-52, projection.hpp:23-31) and run statistics. */
typedef struct pm_run_result {
    char consensus[32];       /* NUL-terminated */
    int32_t score;
    int32_t iterations;
    double expectation;
    uint64_t source_bucket;
    int64_t best_trial;       /* 0 when this shard found no enriched bucket */
    int64_t trials_run;
    int64_t buckets_enriched;
    double wall_ms;
    int32_t k, s;
    int64_t m;
    double q;
    int32_t t_hat;
    int32_t found;            /* 1 if a candidate exists (shards may legitimately have none) */
    /* ---- extensions ---- */
    int32_t within_d;         /* sequences holding an occurrence of `consensus` within d mismatches */
    int32_t total_distance;   /* sum_i min_j hamming(consensus, S_ij)  (oracle.hpp:101-115) */
    double stage_ms[8];       /* profile=1: [0] keys [1] sort [2] enrich [3] em [4] reduce [5] score [6] h2d+encode [7] d2h */
    int64_t gpu_launches;     /* kernels launched by this call */
    int64_t em_lookup_adds;   /* E-step lookup-adds executed: sum over buckets of (iterations+1) * x * l */
    int64_t h2d_bytes;        /* bytes this call copied host->device ... */
    int64_t d2h_bytes;        /* ... and device->host */
    int64_t em_work;          /* SURVEY §8(d) W_EM: sum_b (2 I_b+1) x l + 4 (I_b+1) x  (E- and M-step work) */
    int64_t em_tensor_flops;  /* dense tcgen05.mma FLOPs the tensor-core EM kernel issued (2 M N K per instruction) */
    int64_t em_exact_buckets; /* buckets refined again by the pair kernel (flagged by the tensor-core kernel) ... */
    int64_t em_fp64_buckets;  /* ... and by the FP64 kernel (stop decisions near tol, candidates of near-equal expectation) */
} pm_run_result;

/* --------------------------------------------------------------------------------------------
 * 1. Host-only entry points (no GPU needed)
 * ------------------------------------------------------------------------------------------ */
const char* pm_version(void);
const char* pm_last_error(void);
void pm_default_config(pm_run_config* cfg);                        /* RunConfig{} defaults, driver.hpp:23-42 */

uint64_t pm_splitmix64(uint64_t x);                                /* rng.hpp:13-17 */
uint64_t pm_derive_seed(uint64_t master, uint64_t index);          /* rng.hpp:22-24 */
int pm_sample_plan(int l, int k, uint64_t rng_seed, int32_t* kept);/* sample_plan(l,k,Rng(seed)), projection.hpp:210-226 */
/* sample_plan(l,k,rng) on a generator the CALLER owns (projection.hpp:210-226, rng.hpp:37-73): next_u64(state) must
 * return the generator's next 64-bit output; the l-k draws (plus rejections) are taken from it, so consecutive calls
 * on one generator give the reference's consecutive plans. */
int pm_sample_plan_stream(int l, int k, uint64_t (*next_u64)(void*), void* state, int32_t* kept);
int pm_trial_plan(int l, int k, uint64_t master, int64_t trial, int32_t* kept); /* driver.hpp:164-165 */
int pm_validate_plan(int l, const int32_t* kept, int k);           /* ProjectionPlan ctor, projection.hpp:36-52 */

/* generate_planted, planted.hpp:38-101 (host; the synthetic-input generator of the benchmarks):
 * bases = t*n chars without separators, motif = l chars, positions = t 1-based starts. */
int pm_generate_planted(int t, int n, int l, int d, uint64_t seed, char* bases, char* motif, int32_t* positions);

int pm_optimal_k(int l, int d, int* k);                            /* projection.hpp:97-103 */
int pm_p_hat(int l, int d, int k, double* out);                    /* projection.hpp:107-120 */
int pm_binomial_lt(int t_hat, double p, int s, double* out);       /* projection.hpp:123-148 */
int pm_trials_for_tail(double q, double miss, int64_t* m);         /* projection.hpp:153-174 */
int pm_num_trials(double q, int t_hat, double p, int s, int64_t* m); /* projection.hpp:176-178 */
int pm_bucket_threshold_for_windows(uint64_t windows, int k, int floor_, int* s); /* projection.hpp:182-197 */
/* resolve_params, driver.hpp:55-120; fills k, s, m, q, t_hat of *params. Validates lengths only
 * (symbols are validated on upload, sequence.hpp:44-69). */
int pm_resolve_params(const pm_run_config* cfg, const int64_t* offs, int t, pm_run_result* params);
/* detail::candidate_improves, driver.hpp:127-135 */
int pm_candidate_improves(int score_a, double exp_a, uint64_t key_a, int score_b, double exp_b, uint64_t key_b);
/* Multi-GPU reduction: merges per-shard results (contiguous trial shards in ascending order) exactly
 * as the ascending-trial scan of driver.hpp:195-208 would, including early stop. positions arrays are
 * t ints each (parts_positions[i] may be NULL). Returns PM_ERR_NO_ENRICHED_BUCKETS if no part found one. */
int pm_merge_results(const pm_run_result* parts, const int32_t* const* parts_positions, int n_parts, int t, int l,
                     int early_stop, pm_run_result* out, int32_t* positions_out);

/* --------------------------------------------------------------------------------------------
 * 2. Device context: one per process/GPU.  Holds the 2-bit packed sequence set in HBM.
 * ------------------------------------------------------------------------------------------ */
typedef struct pm_ctx pm_ctx;
/* device: CUDA ordinal; stream: a cudaStream_t (NULL = the legacy default stream). */
int pm_ctx_create(int device, void* stream, pm_ctx** out);
void pm_ctx_destroy(pm_ctx* ctx);
/* SequenceSet ctor (sequence.hpp:44-69) + 2-bit encoding on the device (alphabet.hpp:33-36).
 * Copies the ASCII bases host->device and packs them there; errors: empty set/sequence
 * (InvalidParams), symbol outside ACGT (UnknownSymbol). */
int pm_ctx_set_sequences(pm_ctx* ctx, const char* bases, const int64_t* offs, int t);
/* generate_planted (planted.hpp:38-101) ON THE DEVICE, straight into this context: the reference's mt19937_64 stream
 * (one CTA, 156-way parallel twists) and its contractual draw order, byte-identical to pm_generate_planted for the same
 * seed; the ASCII bases never cross PCIe on the way in.  Optional outputs (NULL to skip): bases_out t*n chars, motif l
 * chars, positions t 1-based starts.  A seed whose stream makes the reference redraw a bounded value (p < 1e-16 per
 * draw) is refused with PM_ERR_UNSUPPORTED rather than generated differently. */
int pm_ctx_generate_planted(pm_ctx* ctx, int t, int n, int l, int d, uint64_t seed, char* bases_out, char* motif,
                            int32_t* positions);
/* Plans of trials first_trial, first_trial + stride, ... (n of them) sampled ON THE DEVICE from the reference's PRNG
 * stream (driver.hpp:164-165, projection.hpp:210-226, rng.hpp:13-73): what pm_run uses for seed-derived plans of sets
 * that take the one-CTA bucketing.  kept: n x k kept positions (1-based, ascending), identical to pm_trial_plan. */
int pm_ctx_trial_plans(pm_ctx* ctx, int l, int k, uint64_t master, int64_t first_trial, int64_t stride, int n, int32_t* kept);
int pm_ctx_num_sequences(const pm_ctx* ctx);
int64_t pm_ctx_total_lmers(const pm_ctx* ctx, int l);               /* sequence.hpp:113-120; <0 if some n_i < l */
int pm_ctx_packed_words(pm_ctx* ctx, uint64_t* words_out, int64_t* word_off_out /* t+1 */, int64_t cap_words);
int pm_ctx_symbol_counts(pm_ctx* ctx, int64_t* counts4);            /* global A,C,T,G counts (refine.hpp:115-125) */
int pm_ctx_synchronize(pm_ctx* ctx);
int64_t pm_ctx_launch_count(const pm_ctx* ctx);                     /* kernels launched so far on this context */
/* EM refinement runs on the tensor cores (128 buckets per CTA, pm_em_tc.cuh).  A bucket whose discrete outputs are not
 * clear of the FP32 error of those sums is refined again by the pair kernel (FP64 on the windows that decide), and a
 * bucket whose stop decision (refine.hpp:300) is within the pair kernel's own likelihood error by the FP64 kernel.
 * out6 = counts of the last pm_refine / pm_run on this context: [0] buckets handed to the pair kernel, then by reason
 * [1] likelihood gain near tol [2] maximum left the exponent range [3] argmax runner-up within delta (refine.hpp:311-316)
 * [4] non-finite weight; [5] buckets handed to the FP64 kernel. */
int pm_ctx_em_exact_counts(const pm_ctx* ctx, int64_t* out6);

/* --------------------------------------------------------------------------------------------
 * 3. Stage-level device entry points (each parity-testable in isolation)
 * ------------------------------------------------------------------------------------------ */
/* project_encode over all x l-mers in lmer_refs order: projection.hpp:243-254, :332-339. */
int pm_hash_keys(pm_ctx* ctx, int l, const int32_t* kept, int k, uint64_t* keys_out /* x */);
/* hash_trial, projection.hpp:319-355: buckets ascending by key, members ascending by flat index.
 * Outputs sized x: bucket_keys/bucket_sizes hold *n_buckets entries, members the x flat indices. */
int pm_hash_trial(pm_ctx* ctx, int l, const int32_t* kept, int k, int backend, uint64_t dense_table_cap,
                  int64_t* n_buckets, uint64_t* bucket_keys, int32_t* bucket_sizes, int32_t* members);
/* hash_trial + enriched_buckets, projection.hpp:359-390: size >= s, ordered by pre-truncation size
 * descending then key ascending, members truncated to r_cap. Outputs sized x (mem_off: x+1). */
int pm_enriched_buckets(pm_ctx* ctx, int l, const int32_t* kept, int k, int s, int r_cap, int64_t* n_enriched,
                        uint64_t* keys, int32_t* sizes_pre, int32_t* overflowed, int64_t* mem_off, int32_t* members);
/* refine, refine.hpp:288-326, for n_buckets member lists at once (bucket b = members[mem_off[b]..mem_off[b+1])).
 * Per bucket: consensus (32 bytes each), positions (t each), score, expectation, iterations,
 * theta (4*(l+1) doubles, MotifModel layout refine.hpp:65-71) and the LL trace (max_iters doubles).
 * Any output pointer may be NULL. */
int pm_refine(pm_ctx* ctx, int l, const int32_t* members, const int64_t* mem_off, int n_buckets, int max_iters,
              double tol, double z_epsilon, char* consensus, int32_t* positions, int32_t* score, double* expectation,
              int32_t* iterations, double* theta, double* ll_trace);
/* The same refinement entirely in FP64, in the reference's own operation order (one CTA per bucket, not a throughput
 * path).  run() uses it to settle candidates of equal score whose expectations differ by less than the FP32 error
 * (detail::candidate_improves compares doubles exactly, driver.hpp:127-135). */
int pm_refine_exact(pm_ctx* ctx, int l, const int32_t* members, const int64_t* mem_off, int n_buckets, int max_iters,
                    double tol, char* consensus, int32_t* positions, int32_t* score, double* expectation,
                    int32_t* iterations, double* theta, double* ll_trace);
/* init_model, refine.hpp:90-127: theta0 (4 x (l+1), MotifModel layout refine.hpp:65-71) of a member list with a
 * pseudocount; the background column holds the symbol frequencies of the whole set.  Errors: empty member list
 * (EmptyBucket), negative pseudocount (InvalidParams). */
int pm_init_model(pm_ctx* ctx, int l, const int32_t* members, int n_members, double pseudocount, double* theta_out);
/* em_step, refine.hpp:216-282: one E-step + M-step from theta_in; *log_likelihood is the OOPS likelihood of theta_in
 * (refine.hpp:209).  pm_em_step runs the production EM kernel (FP32 sums, FP64 normalisation), pm_em_step_exact the FP64
 * kernel. */
int pm_em_step(pm_ctx* ctx, int l, const double* theta_in, double* theta_out, double* log_likelihood);
int pm_em_step_exact(pm_ctx* ctx, int l, const double* theta_in, double* theta_out, double* log_likelihood);
/* expectation, refine.hpp:130-136 (host arithmetic on a 4 x (l+1) model). */
int pm_expectation(const double* theta, int l, double* out);
/* score / consensus of a start vector, scoring.hpp:111-131 (starts 1-based). */
int pm_score(pm_ctx* ctx, int l, const int32_t* starts, int* score, char* consensus /* l+1 */);
/* XOR/popcount Hamming scan of candidate v over every window: per-sequence minimum distance
 * (sequence.hpp:28-38, oracle.hpp:101-115), their sum, and the number of sequences with min <= d. */
int pm_hamming_scan(pm_ctx* ctx, const char* v, int l, int d, int32_t* per_seq_min /* t or NULL */,
                    int* total_distance, int* within_d);
/* median_string, oracle.hpp:120-149: exhaustive search over the 4^l candidates (ascending code order, first
 * minimiser of total_distance wins) with the XOR/popcount scan -- an exact check of a recovered motif for
 * l <= 16. 4^l > limit -> PM_ERR_SEARCH_SPACE_TOO_LARGE (the reference's default limit is 16,777,216 = 4^12);
 * l > 16 within the limit -> PM_ERR_UNSUPPORTED. median: l+1 bytes. */
int pm_median_string(pm_ctx* ctx, int l, uint64_t limit, char* median, int* total_distance);

/* --------------------------------------------------------------------------------------------
 * 4. The whole path: run(), driver.hpp:145-220
 * ------------------------------------------------------------------------------------------ */
/* Sequences already resident (pm_ctx_set_sequences). positions: t ints or NULL.
 * Optional per-trial outputs for trials [trial_begin, trial_end] (each may be NULL):
 * buckets (enriched count), best_score (-1 if none), best_expectation, best_key. */
int pm_run(pm_ctx* ctx, const pm_run_config* cfg, pm_run_result* out, int32_t* positions, int64_t* trial_buckets,
           int32_t* trial_best_score, double* trial_best_expectation, uint64_t* trial_best_key);
/* run() on SEVERAL GPUs of one node (trials are independent, driver.hpp:164: no data-path collective).  One host thread
 * and one context per entry of `devices` (an ordinal may repeat: several contexts share that GPU); each uploads the set
 * and runs its shard of trials 1..m -- contiguous blocks, or round-robin when strided != 0 -- and the per-shard results
 * (a ~300-byte record and the per-trial bucket counts) are merged on the host exactly as the ascending-trial scan of
 * driver.hpp:195-208 would, early stop included.  Same outputs as pm_run_host. */
int pm_run_multi(const int* devices, int n_devices, int strided, const pm_run_config* cfg, const char* bases,
                 const int64_t* offs, int t, pm_run_result* out, int32_t* positions);
/* Same, from host buffers: upload + encode + run + read-back in one call (the e2e path). */
int pm_run_host(pm_ctx* ctx, const pm_run_config* cfg, const char* bases, const int64_t* offs, int t,
                pm_run_result* out, int32_t* positions);

#ifdef __cplusplus
}
#endif
#endif
