"""Parity of the whole path, run() (driver.hpp:145-220), on the GPU: against runs of the unmodified
reference (tests/golden), against the oracle live on small instances, and -- at BASELINE.json's full
sizes -- through size-independent properties."""
import os
import subprocess

import numpy as np
import pytest

from conftest import EXAMPLE_STARTS, EXPECTATION_TOL
from oracle import pmo

pytestmark = pytest.mark.gpu

INT_FIELDS = ("consensus", "score", "iterations", "source_bucket", "best_trial", "trials_run", "buckets_enriched",
              "k", "s", "m", "t_hat", "positions")


def assert_same_result(got, want):
    for f in INT_FIELDS:
        assert got[f] == want[f], (f, got[f], want[f])
    assert abs(got["expectation"] - want["expectation"]) <= EXPECTATION_TOL


def test_runs_match_reference_goldens(ctx, golden, instance):
    for g in golden["run"]:
        ss, _, _ = instance(*g["instance"])
        ctx.set_sequences(ss.bases, ss.offs)
        assert_same_result(ctx.run(**g["cfg"]), g["result"])


def test_per_trial_outcomes_match_reference(ctx, golden, instance):
    ss, _, _ = instance(20, 600, 15, 4, 42)
    ctx.set_sequences(ss.bases, ss.offs)
    r = ctx.run(per_trial=True, l=15, d=4, k=7, s=4, m=16, seed=7, early_stop=0)
    t = golden["trial_outcomes_c1"]
    assert r["trial_buckets"].tolist() == t["buckets"]
    assert r["trial_score"].tolist() == t["score"]
    assert [int(v) for v in r["trial_key"]] == t["key"]
    np.testing.assert_allclose(r["trial_expectation"], t["expectation"], atol=EXPECTATION_TOL, rtol=0)


def test_worked_example_forced_plan(ctx, example, golden):
    # test_driver.cpp:86-102
    r = ctx.run_host(example.bases, example.offs, l=8, d=1, s=4, forced_kept=[1, 2, 3, 6, 7])
    assert_same_result(r, golden["worked"]["run"])
    assert (r["consensus"], r["score"], r["positions"], r["source_bucket"]) == ("ATGCAACT", 53, EXAMPLE_STARTS, 177)
    assert (r["within_d"], r["total_distance"]) == (7, 3)


def test_early_stop_semantics(ctx, best_oracle, instance):
    # test_driver.cpp:104-122: a d=0 plant is perfect at trial 1
    ss, motif, _ = instance(5, 50, 10, 0, 77)
    ctx.set_sequences(ss.bases, ss.offs)
    r = ctx.run(l=10, d=0, seed=5, m=10)
    assert (r["score"], r["consensus"], r["best_trial"], r["trials_run"]) == (50, motif, 1, 1)
    assert_same_result(r, best_oracle.run(ss, l=10, d=0, seed=5, m=10))
    full = ctx.run(l=10, d=0, seed=5, m=10, early_stop=0)
    assert (full["trials_run"], full["score"]) == (10, 50)
    # early stop inside a later batch: trials after the stopping one are discarded as if never run
    r1 = ctx.run(l=10, d=0, seed=5, m=10, batch_trials=3)
    assert (r1["trials_run"], r1["buckets_enriched"]) == (r["trials_run"], r["buckets_enriched"])


def test_errors_mirror_the_reference(pm, ctx, instance, example):
    ss, _, _ = instance(4, 30, 8, 2, 3)
    ctx.set_sequences(ss.bases, ss.offs)
    with pytest.raises(pm.PmError) as e:  # test_driver.cpp:153-161
        ctx.run(l=8, d=2, s=30, m=2)
    assert e.value.kind == "NoEnrichedBucketsError" and "s=30 in 2 trials" in str(e.value)
    ctx.set_sequences(example.bases, example.offs)
    for kw, kind in ((dict(l=5, d=4), "InvalidParamsError"), (dict(l=41, d=1), "InvalidParamsError"),
                     (dict(l=8, d=6, k=1, s=1000), "UnreachableError"), (dict(l=8, d=1, max_em_iters=0), "InvalidParamsError"),
                     (dict(l=12, d=1, k=12, m=1, backend=0), "DenseTableTooLargeError")):
        with pytest.raises(pm.PmError) as e:
            ctx.run(**kw)
        assert e.value.kind == kind, kw


def test_run_matches_oracle_on_small_and_ragged_sets(ctx, best_oracle):
    rng = np.random.default_rng(7)
    for round_ in range(6):
        t = int(rng.integers(3, 9))
        l = int(rng.integers(6, 12))
        ss = pmo.SeqSet.from_strings(["".join(rng.choice(list("ACGT"), int(rng.integers(l + 10, 90)))) for _ in range(t)])
        kw = dict(l=l, d=1, k=l - 3, s=2, m=5, seed=round_, early_stop=0)
        ctx.set_sequences(ss.bases, ss.offs)
        got, want = ctx.run(**kw), best_oracle.run(ss, **kw)
        # candidates of equal score whose expectations are closer than the FP32 error are settled in FP64
        # (pm_refine_exact), so best_trial / source_bucket are the reference's
        assert_same_result(got, want)


def test_run_matches_reference_on_random_sets_through_every_em_tier(pm, best_oracle):
    """run() against the reference on random sets -- larger than the ones above, ragged, 2 ... 24 sequences, l = 7 ... 18,
    thresholds that enrich hundreds of buckets per trial -- with the tensor-core kernel forced on for every batch
    (PM_B200_EM_TC=2), with its default size rule, and with the pair kernel alone (0): best trial, source bucket,
    positions, score, consensus, iterations and the enriched-bucket count are the reference's in all three."""
    import os
    rng = np.random.default_rng(424242)
    cases = []
    for round_ in range(8):
        t = int(rng.integers(2, 25))
        l = int(rng.integers(7, 19))
        strings = ["".join(rng.choice(list("ACGT"), int(rng.integers(l + 40, 360)))) for _ in range(t)]
        k = int(rng.integers(4, min(l - 1, 8) + 1))
        cases.append((pmo.SeqSet.from_strings(strings), dict(l=l, d=2, k=k, s=int(rng.integers(1, 4)), m=4, seed=100 + round_, early_stop=0)))
    for ss, kw in cases:
        want = best_oracle.run(ss, **kw)
        for mode in ("2", "1", "0"):
            os.environ["PM_B200_EM_TC"] = mode
            try:
                with pm.Context(0) as c:
                    c.set_sequences(ss.bases, ss.offs)
                    got = c.run(**kw)
            finally:
                os.environ.pop("PM_B200_EM_TC", None)
            assert_same_result(got, want)


def test_back_to_back_uploads_and_runs(pm, best_oracle):
    """The upload builds the pair kernel's class-group index on a worker thread and run() samples its plans on the
    device, both while other work is in flight: a context that is re-loaded and run over and over (the end-to-end
    loop of bench.py), re-loaded before it ever ran, re-loaded with a large set in between (synchronous index build),
    and destroyed with the build still pending, must give the reference's result every time."""
    rng = np.random.default_rng(5150)
    sets = []
    for _ in range(6):
        t = int(rng.integers(3, 21))
        sets.append(pmo.SeqSet.from_strings(["".join(rng.choice(list("ACGT"), int(rng.integers(60, 500)))) for _ in range(t)]))
    kw = dict(l=9, d=1, k=5, s=2, m=6, seed=11, early_stop=0)
    want = [best_oracle.run(ss, **kw) for ss in sets]
    big = pmo.SeqSet.from_strings(["".join(rng.choice(list("ACGT"), 300)) for _ in range(90)])  # t > 64: large-set path
    want_big = best_oracle.run(big, **dict(kw, m=2))
    with pm.Context(0) as c:
        for round_ in range(3):
            for ss, w in zip(sets, want):
                assert_same_result(c.run_host(ss.bases, ss.offs, **kw), w)
            c.set_sequences(sets[0].bases, sets[0].offs)   # replaced before anything ran on it
            c.set_sequences(big.bases, big.offs)
            assert_same_result(c.run(**dict(kw, m=2)), want_big)
    for ss in sets[:3]:
        with pm.Context(0) as c:
            c.set_sequences(ss.bases, ss.offs)             # destroyed with the index build possibly still running


def test_results_do_not_depend_on_batching_backend_or_workers(ctx, instance):
    # test_driver.cpp:124-151 (workers x backends) plus the GPU build's own knob (batch size)
    ss, _, _ = instance(8, 60, 9, 2, 1234)
    ctx.set_sequences(ss.bases, ss.offs)
    base = ctx.run(l=9, d=2, seed=42)
    for kw in (dict(workers=4), dict(backend=1), dict(batch_trials=1), dict(batch_trials=7)):
        other = ctx.run(l=9, d=2, seed=42, **kw)
        for f in INT_FIELDS + ("expectation",):
            assert other[f] == base[f], (kw, f)


def test_explicit_plans_and_trial_shards(pm, ctx, instance):
    ss, _, _ = instance(12, 120, 8, 1, 5)
    ctx.set_sequences(ss.bases, ss.offs)
    kw = dict(l=8, d=1, k=5, s=3, m=7, seed=3, early_stop=0)
    full = ctx.run(**kw)
    plans = np.array([pm.trial_plan(8, 5, 3, tr) for tr in range(1, 8)], dtype=np.int32)
    via_plans = ctx.run(plans=plans, **dict(kw, seed=999))
    for f in INT_FIELDS + ("expectation",):
        assert via_plans[f] == full[f], f
    # contiguous shards merged by pm_merge_results == the single run (the multi-GPU reduction)
    from paper_1605_06904_b200.sharding import shard_range
    for world in (2, 3, 4):
        parts, poss = [], []
        for rank in range(world):
            b, e = shard_range(7, rank, world)
            try:
                ctx.run(trial_begin=b, trial_end=e, **kw)
            except pm.PmError as err:
                assert err.kind == "NoEnrichedBucketsError"
            parts.append(ctx.last_result)
            poss.append(ctx.last_positions.copy())
        merged, pos = pm.merge_results(parts, poss, ss.t, 8, False)
        assert (merged.consensus.decode(), merged.score, merged.expectation, merged.source_bucket, merged.best_trial,
                merged.trials_run, merged.buckets_enriched) == \
               (full["consensus"], full["score"], full["expectation"], full["source_bucket"], full["best_trial"],
                full["trials_run"], full["buckets_enriched"])
        assert pos.tolist() == full["positions"]


def test_full_size_properties_c1_c2(ctx, port, golden, instance):
    """BASELINE configs at their full trial counts: properties that do not need the slow CPU EM."""
    for key, l, d, m in (((20, 600, 15, 4, 42), 15, 4, 172), ((20, 1000, 16, 5, 42), 16, 5, 1293)):
        ss, motif, planted_pos = instance(*key)
        ctx.set_sequences(ss.bases, ss.offs)
        kw = dict(l=l, d=d, k=7, s=4, m=m, seed=7, early_stop=0)
        r = ctx.run(per_trial=True, **kw)
        assert r["m"] == m == r["trials_run"]
        # enriched-bucket counts of every trial equal the oracle's hashing stage (bit-exact path)
        sample = list(range(1, m + 1)) if m <= 200 else list(range(1, m + 1, 7))
        for tr in sample:
            kept = port.trial_plan(l, 7, 7, tr)
            assert r["trial_buckets"][tr - 1] == len(port.enriched(ss, l, kept, 4, ss.t * 4)), tr
        # score identity (test_scoring.cpp:108-124): score = l*t - sum_i hamming(consensus, row_i)
        rows = [s[p - 1:p - 1 + l] for s, p in zip(ss.strings(), r["positions"])]
        assert r["score"] == l * ss.t - sum(port.hamming(r["consensus"], row) for row in rows)
        assert port.score(ss, l, r["positions"]) == (r["score"], r["consensus"])
        tot, per = port.total_distance(ss, r["consensus"])
        assert (r["total_distance"], r["within_d"]) == (tot, sum(1 for p in per if p <= d))
        # the best trial's candidate is what the oracle refines from that trial's winning bucket
        kept = port.trial_plan(l, 7, 7, r["best_trial"])
        bucket = [e for e in port.enriched(ss, l, kept, 4, ss.t * 4) if e["key"] == r["source_bucket"]][0]
        c = port.refine(ss, l, bucket["members"], bucket["key"])
        assert (c.consensus, c.positions, c.score, c.iterations) == (r["consensus"], r["positions"], r["score"], r["iterations"])
        assert abs(c.expectation - r["expectation"]) <= EXPECTATION_TOL
        if key[1] == 600:
            assert r["consensus"] == motif  # the planted (15,4) motif is recovered within 172 trials
        # running the same trials again in different batch sizes gives the same answer
        r2 = ctx.run(batch_trials=64, **kw)
        assert (r2["consensus"], r2["score"], r2["best_trial"], r2["buckets_enriched"]) == \
               (r["consensus"], r["score"], r["best_trial"], r["buckets_enriched"])


def test_cpp_host_layer(pm):
    """include/projmotif_b200.hpp: the reference's own test cases restated against the C++ layer."""
    exe = "/tmp/pm_host_layer_test"
    subprocess.run(["g++", "-std=c++17", "-O1", "-I" + os.path.join(pm.REPO_DIR, "include"),
                    os.path.join(pm.REPO_DIR, "tests", "cpp", "host_layer_test.cpp"), "-L" + pm.PKG_DIR, "-lpm_b200",
                    "-Wl,-rpath," + pm.PKG_DIR, "-o", exe], check=True)
    out = subprocess.run([exe], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "all checks passed" in out.stdout


def test_run_with_more_than_1024_sequences(ctx, port):
    """t = 1100 short sequences: multi-tile EM with the per-sequence maxima kept in global memory."""
    rng = np.random.default_rng(3)
    strings = ["".join(rng.choice(list("ACGT"), 40)) for _ in range(1100)]
    ss = pmo.SeqSet.from_strings(strings)
    kw = dict(l=10, d=2, k=8, s=6, m=2, seed=5, early_stop=0)
    ctx.set_sequences(ss.bases, ss.offs)
    got = ctx.run(per_trial=True, **kw)
    b, sc, ex, key = port.trial_outcomes(ss, 1, 2, **kw)
    assert got["trial_buckets"].tolist() == b.tolist()
    assert got["trial_score"].tolist() == sc.tolist()
    assert [int(v) for v in got["trial_key"]] == [int(v) for v in key]
    np.testing.assert_allclose(got["trial_expectation"], ex, atol=EXPECTATION_TOL, rtol=0)


def test_large_scale_c5_hashing_and_one_bucket(pm, ctx, port):
    """BASELINE config 5 at full size (t=10,000 x n=1000, (15,4), k=10, s=19): every key and every
    enriched list bit-exact, one bucket's EM against the oracle (a full CPU trial would take hours)."""
    bases, offs, motif, _ = pm.generate_planted(10000, 1000, 15, 4, 42)
    ss = pmo.SeqSet(bases, offs)
    ctx.set_sequences(bases, offs)
    kept = pm.trial_plan(15, 10, 7, 1)
    assert (ctx.hash_keys(15, kept) == port.hash_keys(ss, 15, kept)).all()
    want = port.enriched(ss, 15, kept, 19, 10000 * 19)
    got = ctx.enriched_buckets(15, kept, 19, 10000 * 19)
    assert got == want and len(got) > 5000
    e = want[len(want) // 3]
    a = ctx.refine(15, [e["members"]])[0]
    w = port.refine(ss, 15, e["members"], e["key"])
    assert (a["consensus"], a["score"], a["iterations"], a["positions"]) == (w.consensus, w.score, w.iterations, w.positions)
    assert np.abs(a["theta"] - w.theta).max() <= 1e-4 and abs(a["expectation"] - w.expectation) <= EXPECTATION_TOL


def test_degenerate_shapes_match_oracle(ctx, best_oracle):
    """Edge shapes the reference accepts: one sequence, one window per sequence (n == l), l = 1,
    identity projection (k == l), windows fewer than a warp, s = 1."""
    cases = [
        (["ACGTACGTACGTAAACCC"], dict(l=4, d=1, k=2, s=2, m=3, seed=1, early_stop=0)),
        (["ACGTAC", "ACGTTC", "ACGAAC", "TTGTAC"], dict(l=6, d=1, k=4, s=2, m=4, seed=2, early_stop=0)),   # n == l
        (["ACGT" * 5, "TTGA" * 6, "CCAG" * 4], dict(l=1, d=0, k=1, s=1, m=1, seed=3, early_stop=0)),        # l = 1
        (["ACGTTGCAAGCT" * 3, "ACGTTGCATGCT" * 3, "GGGTTGCAAGCA" * 2], dict(l=8, d=1, k=8, s=2, m=1, seed=4, early_stop=0)),  # k == l
        (["A" * 40, "A" * 35], dict(l=5, d=0, k=3, s=1, m=1, seed=5, early_stop=0)),                       # all windows identical
    ]
    for strings, kw in cases:
        ss = pmo.SeqSet.from_strings(strings)
        ctx.set_sequences(ss.bases, ss.offs)
        got, want = ctx.run(**kw), best_oracle.run(ss, **kw)
        fields = ("consensus", "score", "positions", "iterations", "source_bucket", "best_trial", "trials_run", "buckets_enriched")
        if len(strings) == 1:
            # t = 1: every candidate scores l and many tie on expectation to the last bit, so the
            # reference's own winner depends on rounding noise; compare the rest
            fields = ("score", "trials_run", "buckets_enriched")
            assert best_oracle.score(ss, kw["l"], got["positions"]) == (got["score"], got["consensus"])
        for f in fields:
            assert got[f] == want[f], (strings[0][:12], f, got[f], want[f])
        assert abs(got["expectation"] - want["expectation"]) <= EXPECTATION_TOL


def test_fused_count_and_sort_bucketing_agree(pm, best_oracle, instance):
    """run() buckets each trial with the one-CTA shared-memory histogram kernel (csrc/pm_hash_fused.cuh) when
    the dense table fits one CTA, with the device-wide counting sort (csrc/pm_hash_count.cuh) when it does not and
    4^k <= 2^20, and with the segmented radix sort otherwise; PM_B200_FUSED_HASH=0 with PM_B200_COUNT_HASH=2 / 0
    force the later paths.  Per-trial outcomes must be identical, on the challenge instance and on low-complexity sets whose
    buckets hold hundreds of members (cooperative ordering), whose key space is smaller than the CTA (k <= 4), or
    whose largest bucket exceeds what the counting path orders in shared memory (it then falls back by itself)."""
    import os
    rng = np.random.default_rng(21)
    low = pmo.SeqSet.from_strings(["".join(rng.choice(list("AC"), 150, p=[0.9, 0.1])) for _ in range(6)])
    ragged = pmo.SeqSet.from_strings(["".join(rng.choice(list("ACGT"), int(rng.integers(40, 200)))) for _ in range(9)])
    mono = pmo.SeqSet.from_strings(["".join(rng.choice(list("AC"), 700, p=[0.97, 0.03])) for _ in range(8)])
    cases = [
        (instance(20, 600, 15, 4, 42)[0], dict(l=15, d=4, k=7, s=4, m=6, seed=7, early_stop=0)),
        (low, dict(l=9, d=2, k=6, s=3, m=4, seed=1, early_stop=0)),      # buckets of several hundred members
        (low, dict(l=9, d=2, k=8, s=40, m=3, seed=2, early_stop=0)),     # 4^8 keys, high threshold, r_cap truncation
        (ragged, dict(l=7, d=1, k=3, s=2, m=5, seed=3, early_stop=0)),   # 64 keys < 512 threads
        (ragged, dict(l=6, d=1, k=1, s=1, m=3, seed=4, early_stop=0)),   # 4 keys
        (mono, dict(l=8, d=1, k=4, s=3, m=2, seed=5, early_stop=0)),     # one bucket of > 4096 members
    ]
    modes = {"fused": {}, "count": {"PM_B200_FUSED_HASH": "0", "PM_B200_COUNT_HASH": "2"},
             "sort": {"PM_B200_FUSED_HASH": "0", "PM_B200_COUNT_HASH": "0"}}
    for ss, kw in cases:
        res = {}
        for name, env in modes.items():
            os.environ.update(env)
            try:
                with pm.Context(0) as c:
                    c.set_sequences(ss.bases, ss.offs)
                    res[name] = c.run(per_trial=True, **kw)
            finally:
                for key in env:
                    os.environ.pop(key, None)
        a = res["fused"]
        assert a["gpu_launches"] < res["count"]["gpu_launches"]  # the fused path really ran
        assert res["count"]["gpu_launches"] != res["sort"]["gpu_launches"]
        for name in ("count", "sort"):
            b = res[name]
            for f in INT_FIELDS + ("expectation",):
                assert a[f] == b[f], (kw, name, f)
            for f in ("trial_buckets", "trial_score", "trial_key", "trial_expectation"):
                assert (a[f] == b[f]).all(), (kw, name, f)
        want = best_oracle.run(ss, **kw)
        assert (a["score"], a["buckets_enriched"], a["trials_run"]) == (want["score"], want["buckets_enriched"], want["trials_run"])


def test_large_scale_c5_counting_sort_equals_radix_sort(pm):
    """BASELINE config 5 at full size through run(): one trial with the reference-derived k=10, s=19 (5,346 enriched
    buckets of ~20 members) and one with k=7, s=4 (all 16,384 buckets enriched, ~600 members each: the M-step at
    scale) -- the counting-sort bucketing against the radix-sort path, every per-trial outcome identical."""
    import os
    bases, offs, motif, _ = pm.generate_planted(10000, 1000, 15, 4, 42)
    for k, s, n_enriched in ((10, 19, None), (7, 4, 16384)):
        res = {}
        for flag in ("2", "0"):
            os.environ["PM_B200_COUNT_HASH"] = flag
            try:
                with pm.Context(0) as c:
                    c.set_sequences(bases, offs)
                    res[flag] = c.run(per_trial=True, l=15, d=4, k=k, s=s, m=1, seed=7, early_stop=0)
            finally:
                os.environ.pop("PM_B200_COUNT_HASH", None)
        a, b = res["2"], res["0"]
        for f in INT_FIELDS + ("expectation",):
            assert a[f] == b[f], (k, s, f)
        for f in ("trial_buckets", "trial_score", "trial_key", "trial_expectation"):
            assert (a[f] == b[f]).all(), (k, s, f)
        assert a["buckets_enriched"] > 5000 and (n_enriched is None or a["buckets_enriched"] == n_enriched)
