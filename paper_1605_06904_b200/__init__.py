"""paper_1605_06904_b200 — B200 (sm_100a) implementation of the PROJECTION motif-finding hot path.

The product is the C-ABI shared library ``libpm_b200.so`` (include/pm_b200.h) built from
``csrc/`` with nvcc; the C++ host layer with the reference's own signatures is
include/projmotif_b200.hpp.  This module is the thin ctypes binding that tests/ and bench.py use
to call that ABI; it contains no algorithm and no fallback: if the library is missing or no
sm_100 GPU is present, device calls raise.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import sys

import numpy as np

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
REPO_DIR = os.path.dirname(PKG_DIR)
LIB_PATH = os.environ.get("PM_B200_LIB") or os.path.join(PKG_DIR, "libpm_b200.so")  # override: instrumented builds
CSRC = os.path.join(PKG_DIR, "csrc")
SOURCES = ["pm_capi.cu", "pm_host.cpp"]
HEADERS = ["pm_plans.cuh", "pm_kernels.cuh", "pm_em_smem.cuh", "pm_em_pair.cuh", "pm_em_tc.cuh", "pm_em_f64.cuh", "pm_planted.cuh", "pm_hash_fused.cuh", "pm_hash_count.cuh", "pm_internal.hpp", os.path.join(REPO_DIR, "include", "pm_b200.h")]
NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo", "-O3", "-std=c++17",
              "-Xcompiler", "-fPIC", "-shared"]

STATUS_NAMES = {
    0: "ok", 1: "InvalidParamsError", 2: "LengthMismatchError", 3: "KmerTooLongError",
    4: "DenseTableTooLargeError", 5: "UnreachableError", 6: "EmptyBucketError",
    7: "NoEnrichedBucketsError", 8: "NumericalUnderflowError", 9: "UnknownSymbolError",
    10: "IndexOutOfRangeError", 11: "SearchSpaceTooLargeError", 50: "Unsupported", 100: "CudaError", 101: "NoDevice", 102: "OutOfMemory",
}


class PmError(RuntimeError):
    """A nonzero pm_status; `.kind` is the reference exception name it mirrors (errors.hpp)."""

    def __init__(self, code, msg):
        super().__init__(f"{STATUS_NAMES.get(code, code)}: {msg}")
        self.code = code
        self.kind = STATUS_NAMES.get(code, str(code))


def _nvcc():
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.sep not in cand or os.path.exists(cand)):
            return cand
    return "nvcc"


def needs_build():
    if not os.path.exists(LIB_PATH):
        return True
    built = os.path.getmtime(LIB_PATH)
    deps = [os.path.join(CSRC, s) for s in SOURCES] + [h if os.path.isabs(h) else os.path.join(CSRC, h) for h in HEADERS]
    return any(os.path.getmtime(d) > built for d in deps)


def build(force=False, verbose=False):
    """Compile libpm_b200.so in-tree for sm_100a (nvcc cross-compiles without a GPU)."""
    if not force and not needs_build():
        return LIB_PATH
    cmd = [_nvcc()] + NVCC_FLAGS + ["-o", LIB_PATH] + [os.path.join(CSRC, s) for s in SOURCES]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True)
    return LIB_PATH


class RunConfig(C.Structure):
    """pm_run_config (include/pm_b200.h); mirrors RunConfig, driver.hpp:23-42."""
    _fields_ = [
        ("l", C.c_int32), ("d", C.c_int32), ("k", C.c_int32), ("s", C.c_int32),
        ("m", C.c_int64), ("q", C.c_double), ("seed", C.c_uint64),
        ("workers", C.c_int32), ("backend", C.c_int32), ("max_em_iters", C.c_int32), ("s_floor", C.c_int32),
        ("em_tol", C.c_double), ("dense_table_cap", C.c_uint64),
        ("early_stop", C.c_int32), ("t_hat", C.c_int32),
        ("forced_kept", C.POINTER(C.c_int32)), ("n_forced", C.c_int32), ("_pad0", C.c_int32),
        ("plans", C.POINTER(C.c_int32)), ("trial_begin", C.c_int64), ("trial_end", C.c_int64),
        ("batch_trials", C.c_int32), ("profile", C.c_int32), ("z_epsilon", C.c_double),
        ("trial_stride", C.c_int64), ("exact_best", C.c_int32), ("_pad1", C.c_int32),
    ]


class RunResult(C.Structure):
    """pm_run_result (include/pm_b200.h); mirrors RunResult + TrialParams, driver.hpp:44-52."""
    _fields_ = [
        ("consensus", C.c_char * 32), ("score", C.c_int32), ("iterations", C.c_int32),
        ("expectation", C.c_double), ("source_bucket", C.c_uint64),
        ("best_trial", C.c_int64), ("trials_run", C.c_int64), ("buckets_enriched", C.c_int64),
        ("wall_ms", C.c_double), ("k", C.c_int32), ("s", C.c_int32), ("m", C.c_int64),
        ("q", C.c_double), ("t_hat", C.c_int32), ("found", C.c_int32),
        ("within_d", C.c_int32), ("total_distance", C.c_int32),
        ("stage_ms", C.c_double * 8), ("gpu_launches", C.c_int64), ("em_lookup_adds", C.c_int64),
        ("h2d_bytes", C.c_int64), ("d2h_bytes", C.c_int64), ("em_work", C.c_int64),
        ("em_tensor_flops", C.c_int64), ("em_exact_buckets", C.c_int64), ("em_fp64_buckets", C.c_int64),
    ]

    def as_dict(self):
        d = {name: getattr(self, name) for name, _ in self._fields_ if name not in ("consensus", "stage_ms")}
        d["consensus"] = self.consensus.decode()
        d["stage_ms"] = list(self.stage_ms)
        return d


EXPORTS = [
    "pm_version", "pm_last_error", "pm_default_config", "pm_splitmix64", "pm_derive_seed", "pm_sample_plan",
    "pm_sample_plan_stream", "pm_trial_plan", "pm_validate_plan", "pm_generate_planted", "pm_optimal_k", "pm_p_hat", "pm_binomial_lt", "pm_trials_for_tail",
    "pm_num_trials", "pm_bucket_threshold_for_windows", "pm_resolve_params", "pm_candidate_improves",
    "pm_merge_results", "pm_ctx_create", "pm_ctx_destroy", "pm_ctx_set_sequences", "pm_ctx_generate_planted", "pm_ctx_num_sequences",
    "pm_ctx_trial_plans", "pm_ctx_total_lmers", "pm_ctx_packed_words", "pm_ctx_symbol_counts", "pm_ctx_synchronize",
    "pm_ctx_launch_count", "pm_ctx_em_exact_counts", "pm_hash_keys", "pm_hash_trial", "pm_enriched_buckets", "pm_refine", "pm_refine_exact",
    "pm_init_model", "pm_em_step", "pm_em_step_exact", "pm_expectation", "pm_score",
    "pm_hamming_scan", "pm_median_string", "pm_run", "pm_run_host", "pm_run_multi",
]

_lib = None


def lib():
    """Loads libpm_b200.so; raises if it has not been built (there is no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise FileNotFoundError(
                f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'`; "
                "this package has no CPU or PyTorch fallback")
        L = C.CDLL(LIB_PATH)
        L.pm_version.restype = C.c_char_p
        L.pm_last_error.restype = C.c_char_p
        L.pm_splitmix64.restype = C.c_uint64
        L.pm_splitmix64.argtypes = [C.c_uint64]
        L.pm_derive_seed.restype = C.c_uint64
        L.pm_derive_seed.argtypes = [C.c_uint64, C.c_uint64]
        L.pm_ctx_total_lmers.restype = C.c_int64
        L.pm_ctx_total_lmers.argtypes = [C.c_void_p, C.c_int]
        L.pm_ctx_launch_count.restype = C.c_int64
        L.pm_ctx_launch_count.argtypes = [C.c_void_p]
        L.pm_ctx_destroy.argtypes = [C.c_void_p]
        L.pm_ctx_destroy.restype = None
        L.pm_ctx_create.argtypes = [C.c_int, C.c_void_p, C.POINTER(C.c_void_p)]
        _lib = L
    return _lib


def _check(rc):
    if rc != 0:
        raise PmError(rc, lib().pm_last_error().decode())


def _p(a, ty):
    return a.ctypes.data_as(C.POINTER(ty))


def _i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)


# ------------------------------------------------------------------------------------------------
# host-only entry points
# ------------------------------------------------------------------------------------------------
def default_config(**kw) -> RunConfig:
    cfg = RunConfig()
    lib().pm_default_config(C.byref(cfg))
    keep = []
    for key, val in kw.items():
        if key in ("forced_kept", "plans"):
            if val is not None:
                arr = _i32(val).reshape(-1)
                keep.append(arr)
                setattr(cfg, key, _p(arr, C.c_int32))
                if key == "forced_kept":
                    cfg.n_forced = len(arr)
        else:
            setattr(cfg, key, val)
    cfg._keepalive = keep
    return cfg


def derive_seed(master, index):
    return int(lib().pm_derive_seed(C.c_uint64(master), C.c_uint64(index)))


def splitmix64(x):
    return int(lib().pm_splitmix64(C.c_uint64(x)))


def sample_plan(l, k, rng_seed):
    kept = np.zeros(max(k, 1), dtype=np.int32)
    _check(lib().pm_sample_plan(l, k, C.c_uint64(rng_seed), _p(kept, C.c_int32)))
    return kept[:k].tolist()


def trial_plan(l, k, master, trial):
    kept = np.zeros(max(k, 1), dtype=np.int32)
    _check(lib().pm_trial_plan(l, k, C.c_uint64(master), C.c_int64(trial), _p(kept, C.c_int32)))
    return kept[:k].tolist()


def validate_plan(l, kept):
    k = _i32(kept)
    _check(lib().pm_validate_plan(l, _p(k, C.c_int32), len(k)))


def generate_planted(t, n, l, d, seed):
    """planted.hpp:38-101 -> (bases bytes of t*n chars, offs int64[t+1], motif, positions)."""
    bases = C.create_string_buffer(t * n)
    motif = C.create_string_buffer(l + 1)
    pos = np.zeros(t, dtype=np.int32)
    _check(lib().pm_generate_planted(t, n, l, d, C.c_uint64(seed), bases, motif, _p(pos, C.c_int32)))
    return bases.raw[: t * n], np.arange(t + 1, dtype=np.int64) * n, motif.raw[:l].decode(), pos.tolist()


def optimal_k(l, d):
    out = C.c_int()
    _check(lib().pm_optimal_k(l, d, C.byref(out)))
    return out.value


def p_hat(l, d, k):
    out = C.c_double()
    _check(lib().pm_p_hat(l, d, k, C.byref(out)))
    return out.value


def binomial_lt(t_hat, p, s):
    out = C.c_double()
    _check(lib().pm_binomial_lt(t_hat, C.c_double(p), s, C.byref(out)))
    return out.value


def trials_for_tail(q, miss):
    out = C.c_int64()
    _check(lib().pm_trials_for_tail(C.c_double(q), C.c_double(miss), C.byref(out)))
    return out.value


def num_trials(q, t_hat, p, s):
    out = C.c_int64()
    _check(lib().pm_num_trials(C.c_double(q), t_hat, C.c_double(p), s, C.byref(out)))
    return out.value


def bucket_threshold_for_windows(windows, k, floor=3):
    out = C.c_int()
    _check(lib().pm_bucket_threshold_for_windows(C.c_uint64(windows), k, floor, C.byref(out)))
    return out.value


def resolve_params(offs, **kw):
    cfg = default_config(**kw)
    offs = np.ascontiguousarray(offs, dtype=np.int64)
    out = RunResult()
    _check(lib().pm_resolve_params(C.byref(cfg), _p(offs, C.c_int64), len(offs) - 1, C.byref(out)))
    return dict(k=out.k, s=out.s, m=out.m, q=out.q, t_hat=out.t_hat)


def expectation(theta, l):
    """expectation, refine.hpp:130-136."""
    tin = np.ascontiguousarray(theta, dtype=np.float64).reshape(-1)
    out = C.c_double()
    _check(lib().pm_expectation(_p(tin, C.c_double), l, C.byref(out)))
    return out.value


def run_multi(devices, bases: bytes, offs, strided=False, **kw):
    """pm_run_multi: run() sharded over the CUDA devices listed (an ordinal may repeat); same outputs as Context.run_host."""
    cfg = kw.pop("config", None) or default_config(**kw)
    offs = np.ascontiguousarray(offs, dtype=np.int64)
    devs = _i32(devices)
    out = RunResult()
    pos = np.zeros(len(offs) - 1, dtype=np.int32)
    _check(lib().pm_run_multi(_p(devs, C.c_int32), len(devs), int(bool(strided)), C.byref(cfg), bases, _p(offs, C.c_int64),
                              len(offs) - 1, C.byref(out), _p(pos, C.c_int32)))
    d = out.as_dict()
    d["positions"] = pos.tolist()
    return d


def candidate_improves(a, b):
    """a, b: (score, expectation, key)."""
    return bool(lib().pm_candidate_improves(a[0], C.c_double(a[1]), C.c_uint64(a[2]), b[0], C.c_double(b[1]),
                                            C.c_uint64(b[2])))


def merge_results(parts, positions, t, l, early_stop):
    """parts: list[RunResult]; positions: list[np.ndarray|None]. Returns (RunResult, positions)."""
    n = len(parts)
    arr = (RunResult * n)(*parts)
    pos_arrays = [None if p is None else _i32(p) for p in positions]
    ptrs = (C.POINTER(C.c_int32) * n)(*[
        C.cast(None, C.POINTER(C.c_int32)) if p is None else _p(p, C.c_int32) for p in pos_arrays])
    out = RunResult()
    out_pos = np.zeros(t, dtype=np.int32)
    _check(lib().pm_merge_results(arr, ptrs, n, t, l, int(early_stop), C.byref(out), _p(out_pos, C.c_int32)))
    return out, out_pos


# ------------------------------------------------------------------------------------------------
# device context
# ------------------------------------------------------------------------------------------------
class Context:
    """pm_ctx: one per process/GPU; owns the packed sequence set in HBM."""

    def __init__(self, device=0, stream=0):
        self._h = C.c_void_p()
        _check(lib().pm_ctx_create(int(device), C.c_void_p(int(stream) or None), C.byref(self._h)))
        self.t = 0
        self.offs = None

    def close(self):
        if self._h:
            lib().pm_ctx_destroy(self._h)
            self._h = C.c_void_p()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- sequences
    def set_sequences(self, bases: bytes, offs):
        offs = np.ascontiguousarray(offs, dtype=np.int64)
        _check(lib().pm_ctx_set_sequences(self._h, bases, _p(offs, C.c_int64), len(offs) - 1))
        self.t = len(offs) - 1
        self.offs = offs

    def generate_planted(self, t, n, l, d, seed):
        """pm_ctx_generate_planted: the planted instance is generated on the device and becomes this context's sequence
        set.  Returns (bases, offs, motif, positions) like the host generator."""
        bases = C.create_string_buffer(t * n)
        motif = C.create_string_buffer(l + 1)
        pos = np.zeros(t, dtype=np.int32)
        _check(lib().pm_ctx_generate_planted(self._h, t, n, l, d, C.c_uint64(seed), bases, motif, _p(pos, C.c_int32)))
        self.t = t
        self.offs = np.arange(t + 1, dtype=np.int64) * n
        return bases.raw[: t * n], self.offs, motif.raw[:l].decode(), pos.tolist()

    def total_lmers(self, l):
        return int(lib().pm_ctx_total_lmers(self._h, l))

    def packed_words(self):
        nwords = int(sum((((int(self.offs[i + 1] - self.offs[i]) + 31) // 32 + 2) & ~1) for i in range(self.t)))
        words = np.zeros(nwords, dtype=np.uint64)
        woff = np.zeros(self.t + 1, dtype=np.int64)
        _check(lib().pm_ctx_packed_words(self._h, _p(words, C.c_uint64), _p(woff, C.c_int64), C.c_int64(nwords)))
        return words, woff

    def symbol_counts(self):
        out = np.zeros(4, dtype=np.int64)
        _check(lib().pm_ctx_symbol_counts(self._h, _p(out, C.c_int64)))
        return out.tolist()

    def synchronize(self):
        _check(lib().pm_ctx_synchronize(self._h))

    def launch_count(self):
        return int(lib().pm_ctx_launch_count(self._h))

    def em_exact_counts(self):
        """Buckets of the last refine()/run() that the tensor-core EM kernel handed to the pair kernel (total and by
        reason) and that the pair kernel handed to the FP64 kernel (fp64)."""
        out = np.zeros(6, dtype=np.int64)
        _check(lib().pm_ctx_em_exact_counts(self._h, _p(out, C.c_int64)))
        return dict(zip(("total", "likelihood_gain", "range", "argmax_tie", "non_finite", "fp64"), out.tolist()))

    # ---- stages
    def trial_plans_device(self, l, k, seed, first_trial, n, stride=1):
        """Plans of n trials sampled on the device (pm_ctx_trial_plans): n x k kept positions."""
        kept = np.zeros((n, k), dtype=np.int32)
        _check(lib().pm_ctx_trial_plans(self._h, l, k, C.c_uint64(seed), C.c_int64(first_trial), C.c_int64(stride), n,
                                         _p(kept, C.c_int32)))
        return kept

    def hash_keys(self, l, kept):
        k = _i32(kept)
        x = max(self.total_lmers(l), 1)
        keys = np.zeros(x, dtype=np.uint64)
        _check(lib().pm_hash_keys(self._h, l, _p(k, C.c_int32), len(k), _p(keys, C.c_uint64)))
        return keys[: max(self.total_lmers(l), 0)]

    def hash_trial(self, l, kept, backend=2, dense_cap=65536):
        k = _i32(kept)
        x = max(self.total_lmers(l), 1)
        nb = C.c_int64()
        keys = np.zeros(x, dtype=np.uint64)
        sizes = np.zeros(x, dtype=np.int32)
        members = np.zeros(x, dtype=np.int32)
        _check(lib().pm_hash_trial(self._h, l, _p(k, C.c_int32), len(k), backend, C.c_uint64(dense_cap), C.byref(nb),
                                   _p(keys, C.c_uint64), _p(sizes, C.c_int32), _p(members, C.c_int32)))
        n = nb.value
        return keys[:n].copy(), sizes[:n].copy(), members[: int(sizes[:n].sum())].copy()

    def enriched_buckets(self, l, kept, s, r_cap):
        k = _i32(kept)
        x = max(self.total_lmers(l), 1)
        ne = C.c_int64()
        keys = np.zeros(x, dtype=np.uint64)
        sizes = np.zeros(x, dtype=np.int32)
        over = np.zeros(x, dtype=np.int32)
        moff = np.zeros(x + 1, dtype=np.int64)
        members = np.zeros(x, dtype=np.int32)
        _check(lib().pm_enriched_buckets(self._h, l, _p(k, C.c_int32), len(k), s, r_cap, C.byref(ne),
                                         _p(keys, C.c_uint64), _p(sizes, C.c_int32), _p(over, C.c_int32),
                                         _p(moff, C.c_int64), _p(members, C.c_int32)))
        n = ne.value
        return [dict(key=int(keys[b]), size=int(sizes[b]), overflowed=bool(over[b]),
                     members=members[moff[b]:moff[b + 1]].tolist()) for b in range(n)]

    def refine(self, l, member_lists, max_iters=5, tol=1e-6, z_epsilon=-1.0, exact=False):
        """refine() for a batch of buckets; member_lists: list of lists of flat l-mer indices.
        exact=True runs the FP64 kernel (pm_refine_exact) instead of the production kernels."""
        nb = len(member_lists)
        moff = np.zeros(nb + 1, dtype=np.int64)
        for b, m in enumerate(member_lists):
            moff[b + 1] = moff[b] + len(m)
        members = _i32(np.concatenate([np.asarray(m, dtype=np.int32) for m in member_lists]) if nb else [])
        cons = C.create_string_buffer(32 * max(nb, 1))
        pos = np.zeros((max(nb, 1), self.t), dtype=np.int32)
        score = np.zeros(max(nb, 1), dtype=np.int32)
        exp_ = np.zeros(max(nb, 1), dtype=np.float64)
        its = np.zeros(max(nb, 1), dtype=np.int32)
        theta = np.zeros((max(nb, 1), 4, l + 1), dtype=np.float64)
        ll = np.zeros((max(nb, 1), max_iters), dtype=np.float64)
        if exact:
            _check(lib().pm_refine_exact(self._h, l, _p(members, C.c_int32), _p(moff, C.c_int64), nb, max_iters,
                                         C.c_double(tol), cons, _p(pos, C.c_int32), _p(score, C.c_int32),
                                         _p(exp_, C.c_double), _p(its, C.c_int32), _p(theta, C.c_double), _p(ll, C.c_double)))
        else:
            _check(lib().pm_refine(self._h, l, _p(members, C.c_int32), _p(moff, C.c_int64), nb, max_iters, C.c_double(tol),
                                   C.c_double(z_epsilon), cons, _p(pos, C.c_int32), _p(score, C.c_int32),
                                   _p(exp_, C.c_double), _p(its, C.c_int32), _p(theta, C.c_double), _p(ll, C.c_double)))
        out = []
        for b in range(nb):
            out.append(dict(consensus=cons.raw[32 * b: 32 * b + l].decode(), positions=pos[b].tolist(),
                            score=int(score[b]), expectation=float(exp_[b]), iterations=int(its[b]),
                            theta=theta[b].copy(), ll_trace=ll[b, : int(its[b])].tolist()))
        return out

    def init_model(self, l, members, pseudocount=0.0):
        """init_model, refine.hpp:90-127 -> theta0 as a (4, l+1) array (column 0 = background)."""
        m = _i32(members)
        theta = np.zeros((4, l + 1), dtype=np.float64)
        _check(lib().pm_init_model(self._h, l, _p(m, C.c_int32), len(m), C.c_double(pseudocount), _p(theta, C.c_double)))
        return theta

    def em_step(self, l, theta, exact=False):
        """em_step, refine.hpp:216-282 -> (theta', log-likelihood of theta)."""
        tin = np.ascontiguousarray(theta, dtype=np.float64).reshape(-1)
        tout = np.zeros_like(tin)
        ll = C.c_double()
        fn = lib().pm_em_step_exact if exact else lib().pm_em_step
        _check(fn(self._h, l, _p(tin, C.c_double), _p(tout, C.c_double), C.byref(ll)))
        return tout.reshape(4, l + 1), ll.value

    def score(self, l, starts):
        st = _i32(starts)
        sc = C.c_int()
        cons = C.create_string_buffer(l + 1)
        _check(lib().pm_score(self._h, l, _p(st, C.c_int32), C.byref(sc), cons))
        return sc.value, cons.value.decode()

    def hamming_scan(self, v, d):
        per = np.zeros(self.t, dtype=np.int32)
        tot = C.c_int()
        within = C.c_int()
        _check(lib().pm_hamming_scan(self._h, v.encode(), len(v), d, _p(per, C.c_int32), C.byref(tot), C.byref(within)))
        return per.tolist(), tot.value, within.value

    def median_string(self, l, limit=16777216):
        """median_string, oracle.hpp:120-149, on the device (l <= 16): (median, total_distance)."""
        med = C.create_string_buffer(l + 1)
        dist = C.c_int()
        _check(lib().pm_median_string(self._h, l, C.c_uint64(limit), med, C.byref(dist)))
        return med.value.decode(), dist.value

    # ---- the whole path
    def run(self, per_trial=False, **kw):
        cfg = kw.pop("config", None) or default_config(**kw)
        out = RunResult()
        pos = np.zeros(self.t, dtype=np.int32)
        extra = {}
        if per_trial:
            params = resolve_params(self.offs, **{k: v for k, v in kw.items()})
            tb = cfg.trial_begin or 1
            te = cfg.trial_end or params["m"]
            n = te - tb + 1
            extra = dict(buckets=np.zeros(n, dtype=np.int64), score=np.zeros(n, dtype=np.int32),
                         expectation=np.zeros(n, dtype=np.float64), key=np.zeros(n, dtype=np.uint64))
            rc = lib().pm_run(self._h, C.byref(cfg), C.byref(out), _p(pos, C.c_int32), _p(extra["buckets"], C.c_int64),
                              _p(extra["score"], C.c_int32), _p(extra["expectation"], C.c_double),
                              _p(extra["key"], C.c_uint64))
        else:
            rc = lib().pm_run(self._h, C.byref(cfg), C.byref(out), _p(pos, C.c_int32), None, None, None, None)
        self.last_result = out
        self.last_positions = pos
        _check(rc)
        d = out.as_dict()
        d["positions"] = pos.tolist()
        d.update({"trial_" + k: v for k, v in extra.items()})
        return d

    def run_host(self, bases: bytes, offs, **kw):
        cfg = kw.pop("config", None) or default_config(**kw)
        offs = np.ascontiguousarray(offs, dtype=np.int64)
        out = RunResult()
        pos = np.zeros(len(offs) - 1, dtype=np.int32)
        rc = lib().pm_run_host(self._h, C.byref(cfg), bases, _p(offs, C.c_int64), len(offs) - 1, C.byref(out),
                               _p(pos, C.c_int32))
        self.t = len(offs) - 1
        self.offs = offs
        self.last_result = out
        self.last_positions = pos
        _check(rc)
        d = out.as_dict()
        d["positions"] = pos.tolist()
        return d
