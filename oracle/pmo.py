"""ctypes binding of the oracle C ABI (oracle/pmo.h).

TEST INFRASTRUCTURE ONLY: importable from tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs.  The product package never imports this module.

`load("port")` opens oracle/libpm_oracle.so (plain-C restatement, built by oracle/Makefile),
`load("reference")` opens oracle/_ref/libpm_ref.so (the unmodified reference behind the same ABI;
present only where it was built from /root/reference).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "libpm_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libpm_ref.so")
REFERENCE_ROOT = "/root/reference"

ERR_NAMES = {
    0: "ok", 1: "InvalidParamsError", 2: "LengthMismatchError", 3: "KmerTooLongError",
    4: "DenseTableTooLargeError", 5: "UnreachableError", 6: "EmptyBucketError",
    7: "NoEnrichedBucketsError", 8: "NumericalUnderflowError", 9: "UnknownSymbolError",
    10: "IndexOutOfRangeError", 11: "SearchSpaceTooLargeError", 99: "Error",
}


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{ERR_NAMES.get(code, code)}: {msg}")
        self.code = code
        self.kind = ERR_NAMES.get(code, str(code))


class RunConfigC(C.Structure):
    _fields_ = [
        ("l", C.c_int32), ("d", C.c_int32), ("k", C.c_int32), ("s", C.c_int32),
        ("m", C.c_int64), ("q", C.c_double), ("seed", C.c_uint64),
        ("workers", C.c_int32), ("backend", C.c_int32), ("max_em_iters", C.c_int32), ("s_floor", C.c_int32),
        ("em_tol", C.c_double), ("dense_table_cap", C.c_uint64),
        ("early_stop", C.c_int32), ("t_hat", C.c_int32),
        ("forced_kept", C.POINTER(C.c_int32)), ("n_forced", C.c_int32), ("_pad", C.c_int32),
    ]


class RunResultC(C.Structure):
    _fields_ = [
        ("consensus", C.c_char * 32), ("score", C.c_int32), ("iterations", C.c_int32),
        ("expectation", C.c_double), ("source_bucket", C.c_uint64),
        ("best_trial", C.c_int64), ("trials_run", C.c_int64), ("buckets_enriched", C.c_int64),
        ("wall_ms", C.c_double), ("k", C.c_int32), ("s", C.c_int32), ("m", C.c_int64),
        ("q", C.c_double), ("t_hat", C.c_int32), ("_pad", C.c_int32),
    ]


def build(kind: str = "port") -> str:
    """Compile the requested checker with oracle/Makefile; returns the .so path."""
    target = "all" if kind == "port" else "ref"
    subprocess.run(["make", "-s", "-C", HERE, target], check=True)
    return PORT_SO if kind == "port" else REF_SO


def available(kind: str) -> bool:
    return os.path.exists(PORT_SO if kind == "port" else REF_SO)


@dataclass
class SeqSet:
    """Concatenated ASCII bases + offsets, the layout every C ABI in this repo takes."""
    bases: bytes
    offs: np.ndarray  # int64[t+1]

    @staticmethod
    def from_strings(strings):
        offs = np.zeros(len(strings) + 1, dtype=np.int64)
        for i, s in enumerate(strings):
            offs[i + 1] = offs[i] + len(s)
        return SeqSet("".join(strings).encode("ascii"), offs)

    @property
    def t(self):
        return len(self.offs) - 1

    def strings(self):
        b = self.bases.decode("ascii")
        return [b[self.offs[i]:self.offs[i + 1]] for i in range(self.t)]

    def total_lmers(self, l):
        return int(sum(max(0, int(self.offs[i + 1] - self.offs[i]) - l + 1) for i in range(self.t)))

    def flat_to_ref(self, l, flat):
        """flat 0-based l-mer index -> (seq_index, offset), both 1-based like LmerRef."""
        first = 0
        for i in range(self.t):
            w = int(self.offs[i + 1] - self.offs[i]) - l + 1
            if flat < first + w:
                return (i + 1, flat - first + 1)
            first += w
        raise IndexError(flat)

    def ref_to_flat(self, l, seq_index, offset):
        first = 0
        for i in range(seq_index - 1):
            first += int(self.offs[i + 1] - self.offs[i]) - l + 1
        return first + offset - 1


def _p(a, ty):
    return a.ctypes.data_as(C.POINTER(ty))


@dataclass
class Candidate:
    consensus: str
    positions: list
    score: int
    expectation: float
    iterations: int
    theta: np.ndarray | None = None
    ll_trace: list = field(default_factory=list)


class Oracle:
    def __init__(self, path):
        self.lib = C.CDLL(path)
        L = self.lib
        L.pmo_impl.restype = C.c_char_p
        L.pmo_last_error.restype = C.c_char_p
        L.pmo_splitmix64.restype = C.c_uint64
        L.pmo_splitmix64.argtypes = [C.c_uint64]
        L.pmo_derive_seed.restype = C.c_uint64
        L.pmo_derive_seed.argtypes = [C.c_uint64, C.c_uint64]
        L.pmo_total_lmers.restype = C.c_int64
        self.impl = L.pmo_impl().decode()

    def _check(self, rc):
        if rc != 0:
            raise OracleError(rc, self.lib.pmo_last_error().decode())

    # ---- rng
    def splitmix64(self, x):
        return int(self.lib.pmo_splitmix64(C.c_uint64(x)))

    def derive_seed(self, master, index):
        return int(self.lib.pmo_derive_seed(C.c_uint64(master), C.c_uint64(index)))

    def mt_outputs(self, seed, n):
        out = np.zeros(n, dtype=np.uint64)
        self._check(self.lib.pmo_mt_outputs(C.c_uint64(seed), n, _p(out, C.c_uint64)))
        return out

    def uniform_below(self, seed, bound, n):
        out = np.zeros(n, dtype=np.uint64)
        self._check(self.lib.pmo_uniform_below(C.c_uint64(seed), C.c_uint64(bound), n, _p(out, C.c_uint64)))
        return out

    def sample_plan(self, l, k, rng_seed):
        kept = np.zeros(max(k, 1), dtype=np.int32)
        self._check(self.lib.pmo_sample_plan(l, k, C.c_uint64(rng_seed), _p(kept, C.c_int32)))
        return kept[:k].tolist()

    def sample_plans(self, l, k, rng_seed, n):
        """n consecutive sample_plan calls on ONE Rng(rng_seed)."""
        kept = np.zeros(max(k, 1) * n, dtype=np.int32)
        self._check(self.lib.pmo_sample_plans(l, k, C.c_uint64(rng_seed), n, _p(kept, C.c_int32)))
        return kept.reshape(n, max(k, 1))[:, :k].tolist()

    def trial_plan(self, l, k, master, trial):
        kept = np.zeros(max(k, 1), dtype=np.int32)
        self._check(self.lib.pmo_trial_plan(l, k, C.c_uint64(master), C.c_int64(trial), _p(kept, C.c_int32)))
        return kept[:k].tolist()

    # ---- data
    def generate_planted(self, t, n, l, d, seed):
        bases = C.create_string_buffer(t * n)
        motif = C.create_string_buffer(l + 1)
        pos = np.zeros(t, dtype=np.int32)
        self._check(self.lib.pmo_generate_planted(t, n, l, d, C.c_uint64(seed), bases, motif, _p(pos, C.c_int32)))
        offs = np.arange(t + 1, dtype=np.int64) * n
        return SeqSet(bases.raw[: t * n], offs), motif.raw[:l].decode(), pos.tolist()

    # ---- projection
    def encode_kmer(self, kmer):
        out = C.c_uint64()
        self._check(self.lib.pmo_encode_kmer(kmer.encode(), len(kmer), C.byref(out)))
        return out.value

    def project_encode(self, lmer, kept):
        out = C.c_uint64()
        k = np.asarray(kept, dtype=np.int32)
        self._check(self.lib.pmo_project_encode(lmer.encode(), len(lmer), _p(k, C.c_int32), len(k), C.byref(out)))
        return out.value

    def hash_keys(self, ss: SeqSet, l, kept):
        x = ss.total_lmers(l)
        keys = np.zeros(max(x, 1), dtype=np.uint64)
        k = np.asarray(kept, dtype=np.int32)
        self._check(self.lib.pmo_hash_keys(ss.bases, _p(ss.offs, C.c_int64), ss.t, l, _p(k, C.c_int32), len(k),
                                           _p(keys, C.c_uint64)))
        return keys[:x]

    def hash_trial(self, ss: SeqSet, l, kept, backend=2, dense_cap=65536):
        x = max(ss.total_lmers(l), 1)
        nb = C.c_int64()
        keys = np.zeros(x, dtype=np.uint64)
        sizes = np.zeros(x, dtype=np.int32)
        members = np.zeros(x, dtype=np.int32)
        k = np.asarray(kept, dtype=np.int32)
        self._check(self.lib.pmo_hash_trial(ss.bases, _p(ss.offs, C.c_int64), ss.t, l, _p(k, C.c_int32), len(k),
                                            backend, C.c_uint64(dense_cap), C.byref(nb), _p(keys, C.c_uint64),
                                            _p(sizes, C.c_int32), _p(members, C.c_int32)))
        n = nb.value
        return keys[:n].copy(), sizes[:n].copy(), members[: int(sizes[:n].sum())].copy()

    def enriched(self, ss: SeqSet, l, kept, s, r_cap):
        x = max(ss.total_lmers(l), 1)
        ne = C.c_int64()
        keys = np.zeros(x, dtype=np.uint64)
        sizes = np.zeros(x, dtype=np.int32)
        over = np.zeros(x, dtype=np.int32)
        moff = np.zeros(x + 1, dtype=np.int64)
        members = np.zeros(x, dtype=np.int32)
        k = np.asarray(kept, dtype=np.int32)
        self._check(self.lib.pmo_enriched(ss.bases, _p(ss.offs, C.c_int64), ss.t, l, _p(k, C.c_int32), len(k), s,
                                          r_cap, C.byref(ne), _p(keys, C.c_uint64), _p(sizes, C.c_int32),
                                          _p(over, C.c_int32), _p(moff, C.c_int64), _p(members, C.c_int32)))
        n = ne.value
        return [
            dict(key=int(keys[b]), size=int(sizes[b]), overflowed=bool(over[b]),
                 members=members[moff[b]:moff[b + 1]].tolist())
            for b in range(n)
        ]

    # ---- formulas
    def optimal_k(self, l, d):
        out = C.c_int()
        self._check(self.lib.pmo_optimal_k(l, d, C.byref(out)))
        return out.value

    def p_hat(self, l, d, k):
        out = C.c_double()
        self._check(self.lib.pmo_p_hat(l, d, k, C.byref(out)))
        return out.value

    def binomial_lt(self, t_hat, p, s):
        out = C.c_double()
        self._check(self.lib.pmo_binomial_lt(t_hat, C.c_double(p), s, C.byref(out)))
        return out.value

    def trials_for_tail(self, q, miss):
        out = C.c_int64()
        self._check(self.lib.pmo_trials_for_tail(C.c_double(q), C.c_double(miss), C.byref(out)))
        return out.value

    def num_trials(self, q, t_hat, p, s):
        out = C.c_int64()
        self._check(self.lib.pmo_num_trials(C.c_double(q), t_hat, C.c_double(p), s, C.byref(out)))
        return out.value

    def bucket_threshold_for_windows(self, windows, k, floor=3):
        out = C.c_int()
        self._check(self.lib.pmo_bucket_threshold_for_windows(C.c_uint64(windows), k, floor, C.byref(out)))
        return out.value

    # ---- refine
    def init_model(self, ss, l, members, pseudocount=0.0):
        theta = np.zeros(4 * (l + 1), dtype=np.float64)
        m = np.asarray(members, dtype=np.int32)
        self._check(self.lib.pmo_init_model(ss.bases, _p(ss.offs, C.c_int64), ss.t, l, _p(m, C.c_int32), len(m),
                                            C.c_double(pseudocount), _p(theta, C.c_double)))
        return theta.reshape(4, l + 1)

    def em_step(self, ss, l, theta):
        tin = np.ascontiguousarray(theta, dtype=np.float64).reshape(-1)
        tout = np.zeros_like(tin)
        ll = C.c_double()
        self._check(self.lib.pmo_em_step(ss.bases, _p(ss.offs, C.c_int64), ss.t, l, _p(tin, C.c_double),
                                         _p(tout, C.c_double), C.byref(ll)))
        return tout.reshape(4, l + 1), ll.value

    def expectation(self, theta, l):
        tin = np.ascontiguousarray(theta, dtype=np.float64).reshape(-1)
        out = C.c_double()
        self._check(self.lib.pmo_expectation(_p(tin, C.c_double), l, C.byref(out)))
        return out.value

    def refine(self, ss, l, members, key=0, max_iters=5, tol=1e-6, want_theta=True) -> Candidate:
        m = np.asarray(members, dtype=np.int32)
        cons = C.create_string_buffer(l + 1)
        pos = np.zeros(ss.t, dtype=np.int32)
        score = C.c_int()
        exp_ = C.c_double()
        its = C.c_int()
        theta = np.zeros(4 * (l + 1), dtype=np.float64)
        lls = np.full(max(max_iters, 1), np.nan, dtype=np.float64)
        self._check(self.lib.pmo_refine(ss.bases, _p(ss.offs, C.c_int64), ss.t, l, _p(m, C.c_int32), len(m),
                                        C.c_uint64(key), max_iters, C.c_double(tol), cons, _p(pos, C.c_int32),
                                        C.byref(score), C.byref(exp_), C.byref(its),
                                        _p(theta, C.c_double) if want_theta else None,
                                        _p(lls, C.c_double) if want_theta else None))
        return Candidate(cons.value.decode(), pos.tolist(), score.value, exp_.value, its.value,
                         theta.reshape(4, l + 1) if want_theta else None,
                         [float(v) for v in lls[: its.value]] if want_theta else [])

    # ---- scoring
    def score(self, ss, l, starts):
        st = np.asarray(starts, dtype=np.int32)
        sc = C.c_int()
        cons = C.create_string_buffer(l + 1)
        self._check(self.lib.pmo_score(ss.bases, _p(ss.offs, C.c_int64), ss.t, l, _p(st, C.c_int32), C.byref(sc), cons))
        return sc.value, cons.value.decode()

    def hamming(self, a, b):
        out = C.c_int()
        self._check(self.lib.pmo_hamming(a.encode(), b.encode(), len(a), C.byref(out)))
        return out.value

    def total_distance(self, ss, v):
        tot = C.c_int()
        per = np.zeros(ss.t, dtype=np.int32)
        self._check(self.lib.pmo_total_distance(ss.bases, _p(ss.offs, C.c_int64), ss.t, v.encode(), len(v),
                                                C.byref(tot), _p(per, C.c_int32)))
        return tot.value, per.tolist()

    # ---- exact solvers for small instances (oracle.hpp)
    def median_string(self, ss, l, limit=16777216):
        med = C.create_string_buffer(l + 1)
        dist = C.c_int()
        self._check(self.lib.pmo_median_string(ss.bases, _p(ss.offs, C.c_int64), ss.t, l, C.c_uint64(limit), med, C.byref(dist)))
        return med.value.decode(), dist.value

    def naive_mfp(self, ss, l, limit=100000000):
        pos = np.zeros(ss.t, dtype=np.int32)
        sc = C.c_int()
        cons = C.create_string_buffer(l + 1)
        self._check(self.lib.pmo_naive_mfp(ss.bases, _p(ss.offs, C.c_int64), ss.t, l, C.c_uint64(limit), _p(pos, C.c_int32),
                                           C.byref(sc), cons))
        return pos.tolist(), sc.value, cons.value.decode()

    # ---- driver
    def config(self, **kw):
        cfg = RunConfigC()
        self.lib.pmo_default_config(C.byref(cfg))
        keep = None
        for key, val in kw.items():
            if key == "forced_kept":
                if val is not None:
                    keep = np.asarray(val, dtype=np.int32)
                    cfg.forced_kept = _p(keep, C.c_int32)
                    cfg.n_forced = len(keep)
            else:
                setattr(cfg, key, val)
        cfg._keepalive = keep
        return cfg

    def resolve_params(self, ss, **kw):
        cfg = self.config(**kw)
        out = RunResultC()
        self._check(self.lib.pmo_resolve_params(C.byref(cfg), ss.bases, _p(ss.offs, C.c_int64), ss.t, C.byref(out)))
        return dict(k=out.k, s=out.s, m=out.m, q=out.q, t_hat=out.t_hat)

    def run(self, ss, **kw):
        cfg = self.config(**kw)
        out = RunResultC()
        pos = np.zeros(ss.t, dtype=np.int32)
        self._check(self.lib.pmo_run(C.byref(cfg), ss.bases, _p(ss.offs, C.c_int64), ss.t, C.byref(out),
                                     _p(pos, C.c_int32)))
        return dict(consensus=out.consensus.decode(), score=out.score, iterations=out.iterations,
                    expectation=out.expectation, source_bucket=out.source_bucket, best_trial=out.best_trial,
                    trials_run=out.trials_run, buckets_enriched=out.buckets_enriched, wall_ms=out.wall_ms,
                    k=out.k, s=out.s, m=out.m, q=out.q, t_hat=out.t_hat, positions=pos.tolist())

    def trial_outcomes(self, ss, trial_begin, trial_end, **kw):
        cfg = self.config(**kw)
        n = trial_end - trial_begin + 1
        buckets = np.zeros(n, dtype=np.int64)
        score = np.zeros(n, dtype=np.int32)
        exp_ = np.zeros(n, dtype=np.float64)
        key = np.zeros(n, dtype=np.uint64)
        self._check(self.lib.pmo_trial_outcomes(C.byref(cfg), ss.bases, _p(ss.offs, C.c_int64), ss.t,
                                                C.c_int64(trial_begin), C.c_int64(trial_end), _p(buckets, C.c_int64),
                                                _p(score, C.c_int32), _p(exp_, C.c_double), _p(key, C.c_uint64)))
        return buckets, score, exp_, key


def load(kind: str = "port") -> Oracle:
    path = PORT_SO if kind == "port" else REF_SO
    if not os.path.exists(path):
        if kind == "port" or os.path.isdir(os.path.join(REFERENCE_ROOT, "proj", "include", "projmotif")):
            build(kind)
    if not os.path.exists(path):
        raise FileNotFoundError(path)
    return Oracle(path)
