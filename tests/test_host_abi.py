"""CPU-side checks of libpm_b200.so: it loads without a GPU, exports every symbol that
include/pm_b200.h declares, its host logic (plan PRNG stream, formulas, resolve_params, merge)
equals the reference's, and device entry points fail loudly instead of falling back."""
import ctypes as C
import os
import subprocess
import re

import numpy as np
import pytest

from oracle import pmo


def test_library_exports_every_declared_symbol(pm):
    header = open(os.path.join(pm.REPO_DIR, "include", "pm_b200.h")).read()
    declared = set(re.findall(r"\b(pm_[a-z0-9_]+)\s*\(", header))
    declared -= {"pm_status"}
    assert declared == set(pm.EXPORTS), declared ^ set(pm.EXPORTS)
    L = pm.lib()
    for name in declared:
        assert hasattr(L, name), name
    assert b"sm_100a" in L.pm_version()


def test_struct_layouts_match_header(pm):
    # sizes computed from the header's field lists (natural alignment, LP64)
    assert C.sizeof(pm.RunConfig) == 16 + 8 + 8 + 8 + 16 + 8 + 8 + 8 + 8 + 8 + 8 + 8 + 8 + 8 + 8 + 8 + 8  # + trial_stride, exact_best
    assert C.sizeof(pm.RunResult) == 32 + 8 + 8 + 8 + 24 + 8 + 8 + 8 + 8 + 8 + 8 + 64 + 16 + 16 + 8 + 24


def test_no_gpu_means_loud_failure_not_fallback(pm):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present; this test is for the CPU-only container")
    with pytest.raises(pm.PmError) as e:
        pm.Context(0)
    assert e.value.kind == "NoDevice"
    assert "no CPU fallback" in str(e.value)


def test_product_never_touches_the_oracle(pm):
    src_dir = os.path.join(pm.PKG_DIR)
    for root, _, files in os.walk(src_dir):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".hpp", ".h")):
                text = open(os.path.join(root, f)).read()
                assert "pmo_" not in text and "libpm_oracle" not in text and "libpm_ref" not in text, f
                assert not re.search(r"^\s*(from|import)\s+oracle", text, re.M), f


def test_plan_stream_matches_reference(pm, golden, port):
    for m, i, v in golden["derive_seed"]:
        assert pm.derive_seed(m, i) == v
    for p in golden["plans"]:
        assert pm.trial_plan(p["l"], p["k"], p["master"], p["trial"]) == p["kept"]
    for seed in range(50):  # sample_plan properties, test_projection.cpp:116-143
        l = 4 + seed % 20
        k = 1 + seed % l
        kept = pm.sample_plan(l, k, seed)
        assert kept == port.sample_plan(l, k, seed)
        assert len(kept) == k and all(1 <= a < b <= l for a, b in zip(kept, kept[1:])) and 1 <= kept[0] <= l
    assert pm.sample_plan(9, 9, 3) == list(range(1, 10))  # identity plan, zero draws
    # the library draws from an on-demand mt19937_64 (first 156 outputs straight from the seed chain, the
    # standard engine beyond): same stream as the oracle's std::mt19937_64 on both sides of that boundary
    def plan_from_stream(l, k, seed):  # rng.hpp:37-73 + projection.hpp:214-225 over the oracle's raw mt19937_64 outputs
        stream = iter(int(v) for v in port.mt_outputs(seed, l + 64))
        pool = list(range(1, l + 1))
        for i in range(l - k):
            n = l - i
            low_tail = (2 ** 64 - n) % n
            x = next(stream)
            while x < low_tail:
                x = next(stream)
            j = i + (x % n if n > 1 else 0)
            pool[i], pool[j] = pool[j], pool[i]
        return sorted(set(range(1, l + 1)) - set(pool[: l - k]))

    for seed, l, k in ((1, 31, 1), (2, 64, 3), (3, 150, 2), (4, 157, 1), (5, 158, 1), (6, 200, 10), (7, 400, 5),
                       (2 ** 64 - 1, 160, 1), (0, 156, 1)):
        assert pm.sample_plan(l, k, seed) == plan_from_stream(l, k, seed), (seed, l, k)
    assert plan_from_stream(20, 7, 11) == port.sample_plan(20, 7, 11)
    for trial in range(1, 400):
        assert pm.trial_plan(15, 7, 7, trial) == port.trial_plan(15, 7, 7, trial)
    for bad in ((8, []), (8, [0, 1]), (8, [1, 9]), (8, [2, 2]), (8, [3, 2])):
        with pytest.raises(pm.PmError) as e:
            pm.validate_plan(*bad)
        assert e.value.kind == "InvalidParamsError"


def test_cpp_rng_consumes_its_stream(pm, golden):
    """include/projmotif_b200.hpp: Rng is a real std::mt19937_64 and sample_plan(l, k, rng) draws from it, so two calls
    on one Rng give two different plans -- the reference's consecutive plans (host-only: no GPU needed)."""
    exe = "/tmp/pm_rng_test"
    subprocess.run(["g++", "-std=c++17", "-O1", "-I" + os.path.join(pm.REPO_DIR, "include"),
                    os.path.join(pm.REPO_DIR, "tests", "cpp", "rng_test.cpp"), "-L" + pm.PKG_DIR, "-lpm_b200",
                    "-Wl,-rpath," + pm.PKG_DIR, "-o", exe], check=True)
    for e in golden["plans_consecutive"]:
        out = subprocess.run([exe, str(e["l"]), str(e["k"]), str(e["seed"]), str(len(e["plans"]))], capture_output=True, text=True)
        assert out.returncode == 0, (out.returncode, out.stdout, out.stderr)
        lines = out.stdout.strip().split("\n")
        assert lines[-1] == "rng ok"
        assert [[int(v) for v in ln.split()] for ln in lines[:-1]] == e["plans"]
        if e["k"] < e["l"]:
            assert e["plans"][0] != e["plans"][1]


def test_planted_generator_matches_reference(pm, golden):
    import hashlib
    for p in golden["planted"]:
        bases, offs, motif, pos = pm.generate_planted(p["t"], p["n"], p["l"], p["d"], p["seed"])
        assert (motif, pos, hashlib.sha256(bases).hexdigest()) == (p["motif"], p["positions"], p["sha256"])
        assert offs.tolist() == [i * p["n"] for i in range(p["t"] + 1)]
    for bad in ((0, 10, 3, 1), (2, 10, 11, 1), (2, 10, 3, 3)):
        with pytest.raises(pm.PmError) as e:
            pm.generate_planted(*bad, 1)
        assert e.value.kind == "InvalidParamsError"


def test_formulas_match_reference(pm, golden):
    for l, d, k, v in golden["p_hat"]:
        assert pm.p_hat(l, d, k) == v
    for t, p, s, v in golden["binomial_lt"]:
        assert pm.binomial_lt(t, p, s) == v
    for l, d, m in golden["num_trials"]:
        assert pm.num_trials(0.95, 20, pm.p_hat(l, d, 7), 4) == m
    for w, k, f, s in golden["bucket_threshold"]:
        assert pm.bucket_threshold_for_windows(w, k, f) == s
    assert pm.optimal_k(15, 4) == 10
    with pytest.raises(pm.PmError):
        pm.optimal_k(5, 4)
    with pytest.raises(pm.PmError) as e:
        pm.trials_for_tail(0.95, 1.0)
    assert e.value.kind == "UnreachableError"


def test_resolve_params_matches_oracle(pm, port, example):
    offs600 = np.arange(21, dtype=np.int64) * 600
    assert pm.resolve_params(offs600, l=15, d=4) == port.resolve_params(pmo.SeqSet(b"A" * 12000, offs600), l=15, d=4)
    assert pm.resolve_params(offs600, l=15, d=4, k=7, s=4)["m"] == 172
    cases = [dict(l=8, d=1), dict(l=8, d=1, k=5, s=4, m=9), dict(l=8, d=1, forced_kept=[1, 2, 3, 6, 7]),
             dict(l=8, d=1, t_hat=3), dict(l=8, d=2, s_floor=5)]
    for kw in cases:
        assert pm.resolve_params(example.offs, **kw) == port.resolve_params(example, **kw), kw
    errors = [(dict(l=5, d=4), "InvalidParamsError"), (dict(l=8, d=1, q=1.0), "InvalidParamsError"),
              (dict(l=8, d=8), "InvalidParamsError"), (dict(l=41, d=1), "InvalidParamsError"), (dict(l=0, d=0), "InvalidParamsError"),
              (dict(l=8, d=1, t_hat=8), "InvalidParamsError"), (dict(l=8, d=1, k=9), "InvalidParamsError"),
              (dict(l=8, d=1, k=4, forced_kept=[1, 2, 3, 6, 7]), "InvalidParamsError"),
              (dict(l=8, d=1, s=-1), "InvalidParamsError"), (dict(l=8, d=1, m=-1), "InvalidParamsError"),
              (dict(l=8, d=1, s_floor=0), "InvalidParamsError"), (dict(l=8, d=6, k=1, s=1000), "UnreachableError")]
    for kw, kind in errors:
        with pytest.raises(pm.PmError) as e:
            pm.resolve_params(example.offs, **kw)
        assert e.value.kind == kind, kw
        with pytest.raises(pmo.OracleError) as eo:
            port.resolve_params(example, **kw)
        assert eo.value.kind == kind, kw
    with pytest.raises(pm.PmError) as e:
        pm.resolve_params(example.offs, l=8, d=6, k=1, s=1000)
    assert "lower s or k" in str(e.value)


def test_candidate_ordering(pm):
    # driver.hpp:127-135
    assert pm.candidate_improves((10, 1.0, 5), (9, 9.0, 1))
    assert not pm.candidate_improves((9, 9.0, 1), (10, 1.0, 5))
    assert pm.candidate_improves((10, 2.0, 5), (10, 1.0, 1))
    assert pm.candidate_improves((10, 1.0, 1), (10, 1.0, 5))
    assert not pm.candidate_improves((10, 1.0, 5), (10, 1.0, 5))


def _part(pm, score, exp_, key, best_trial, trials_run, buckets, found=1, cons=b"ACGT"):
    r = pm.RunResult()
    r.consensus = cons
    r.score, r.expectation, r.source_bucket = score, exp_, key
    r.best_trial, r.trials_run, r.buckets_enriched, r.found = best_trial, trials_run, buckets, found
    r.k, r.s, r.m, r.q, r.t_hat = 2, 3, 40, 0.95, 4
    return r


def test_merge_results_is_the_ascending_trial_scan(pm):
    t, l = 4, 4
    a = _part(pm, 12, 3.0, 7, 3, 10, 50)
    b = _part(pm, 12, 3.0, 7, 14, 20, 60, cons=b"TTTT")  # exact tie: the earlier shard wins
    c = _part(pm, 13, 1.0, 9, 25, 30, 70, cons=b"GGGG")
    d = _part(pm, 0, 0.0, 0, 0, 40, 0, found=0)
    out, pos = pm.merge_results([a, b, c, d], [np.full(t, 1), np.full(t, 2), np.full(t, 3), None], t, l, False)
    assert (out.consensus, out.score, out.best_trial, out.trials_run, out.buckets_enriched) == (b"GGGG", 13, 25, 40, 180)
    assert pos.tolist() == [3] * t
    out, pos = pm.merge_results([a, b], [np.full(t, 1), np.full(t, 2)], t, l, False)
    assert (out.consensus, out.best_trial) == (b"ACGT", 3) and pos.tolist() == [1] * t
    # early stop: shard b reached the perfect score l*t at its trial 14 and truncated itself there
    b2 = _part(pm, 16, 4.0, 7, 14, 14, 33, cons=b"TTTT")
    out, _ = pm.merge_results([a, b2, c], [None, None, None], t, l, True)
    assert (out.score, out.best_trial, out.trials_run, out.buckets_enriched) == (16, 14, 14, 83)
    with pytest.raises(pm.PmError) as e:
        pm.merge_results([d], [None], t, l, False)
    assert e.value.kind == "NoEnrichedBucketsError"


def test_shard_ranges_partition_the_trials(pm):
    from paper_1605_06904_b200.sharding import shard_range
    for m in (1, 2, 7, 8, 172, 3421):
        for world in (1, 2, 4, 8):
            covered = []
            for r in range(world):
                b, e = shard_range(m, r, world)
                covered += list(range(b, e + 1))
            assert covered == list(range(1, m + 1))
