"""Parity of each CUDA stage (through the C ABI) against the CPU oracle and the reference-generated
goldens: bit-exact for codes, keys, grouping, enriched lists, positions, scores; theta and
expectation within the stated FP32 tolerance (conftest.THETA_TOL / EXPECTATION_TOL)."""
import os

import numpy as np
import pytest

from conftest import EXAMPLE_STARTS, EXPECTATION_TOL, THETA_TOL, sha
from oracle import pmo

pytestmark = pytest.mark.gpu

CODE = {"A": 0, "C": 1, "T": 2, "G": 3}


def random_set(rng, t, lo, hi):
    return pmo.SeqSet.from_strings(["".join(rng.choice(list("ACGT"), int(rng.integers(lo, hi + 1)))) for _ in range(t)])


def pack_reference(strings):
    """DESIGN.md §3 layout restated in Python: base p at bits [62-2(p%32), 64-2(p%32)) of word p/32."""
    words, woff = [], [0]
    for s in strings:
        nw = ((len(s) + 31) // 32 + 2) & ~1  # zero pad word, even count (16-byte aligned sequences for TMA)
        for w in range(nw):
            v = 0
            for p in range(32):
                if w * 32 + p < len(s):
                    v |= CODE[s[w * 32 + p]] << (62 - 2 * p)
            words.append(v)
        woff.append(woff[-1] + nw)
    return words, woff


def test_encode_packs_two_bits_per_base(ctx):
    rng = np.random.default_rng(1)
    for ss in (random_set(rng, 5, 1, 70), random_set(rng, 3, 32, 32), random_set(rng, 9, 63, 130)):
        ctx.set_sequences(ss.bases, ss.offs)
        words, woff = ctx.packed_words()
        want_words, want_off = pack_reference(ss.strings())
        assert woff.tolist() == want_off
        assert [int(w) for w in words] == want_words
        full = ss.bases.decode()
        assert ctx.symbol_counts() == [full.count(c) for c in "ACTG"]


def test_encode_rejects_what_the_reference_rejects(pm, ctx):
    # sequence.hpp:44-69
    for strings, kind in ((["ACGT", "ACNT"], "UnknownSymbolError"), (["acgt"], "UnknownSymbolError"),
                          (["ACGT", ""], "InvalidParamsError")):
        ss = pmo.SeqSet.from_strings(strings)
        with pytest.raises(pm.PmError) as e:
            ctx.set_sequences(ss.bases, ss.offs)
        assert e.value.kind == kind
    with pytest.raises(pm.PmError) as e:
        ctx.set_sequences(b"", np.zeros(1, dtype=np.int64))
    assert e.value.kind == "InvalidParamsError"


def test_hash_keys_match_oracle_on_ragged_random_sets(ctx, best_oracle):
    rng = np.random.default_rng(2)
    for round_ in range(30):
        l = int(rng.integers(1, 32))
        k = int(rng.integers(1, l + 1))
        ss = random_set(rng, int(rng.integers(1, 9)), l, l + 90)
        kept = best_oracle.sample_plan(l, k, round_)
        ctx.set_sequences(ss.bases, ss.offs)
        got = ctx.hash_keys(l, kept)
        want = best_oracle.hash_keys(ss, l, kept)
        assert got.shape == want.shape and (got == want).all(), (l, k, kept)


def test_worked_example_bucket(ctx, example, golden):
    # test_projection.cpp:171-197 + the reference-generated grouping
    w = golden["worked"]
    ctx.set_sequences(example.bases, example.offs)
    keys, sizes, members = ctx.hash_trial(8, w["kept"])
    assert (keys.tolist(), sizes.tolist(), members.tolist()) == (w["keys"], w["sizes"], w["members"])
    b = keys.tolist().index(177)
    start = int(sizes[:b].sum())
    assert [example.flat_to_ref(8, int(f)) for f in members[start:start + sizes[b]]] == \
        [(1, 8), (2, 19), (3, 3), (4, 5), (5, 31), (6, 27), (7, 15)]
    assert ctx.enriched_buckets(8, w["kept"], 4, 28) == w["enriched_s4"]
    assert ctx.enriched_buckets(8, w["kept"], 4, 5) == w["enriched_s4_cap5"]
    assert ctx.enriched_buckets(8, w["kept"], 1, 7 * 33) == w["enriched_s1"]
    assert ctx.enriched_buckets(8, w["kept"], 1000, 1000) == []
    assert list(ctx.score(8, EXAMPLE_STARTS)) == w["score"]
    per, tot, within = ctx.hamming_scan("ATGCAACT", 1)
    assert [tot, per] == w["total_distance"] and within == 7


def test_hash_trial_and_enrichment_match_oracle_random(ctx, best_oracle):
    # dense == grouped == device on random instances (test_projection.cpp:199-227)
    rng = np.random.default_rng(41)
    for round_ in range(40):
        t = int(rng.integers(2, 7))
        l = int(rng.integers(4, 11))
        k = int(rng.integers(1, min(8, l) + 1))
        ss = random_set(rng, t, max(12, l), 30)
        kept = best_oracle.sample_plan(l, k, round_)
        ctx.set_sequences(ss.bases, ss.offs)
        got = ctx.hash_trial(l, kept)
        for backend in (0, 1):
            want = best_oracle.hash_trial(ss, l, kept, backend)
            assert all((a == b).all() for a, b in zip(got, want))
        for s, r_cap in ((1, 3), (2, 2 * t), (3, 3)):
            assert ctx.enriched_buckets(l, kept, s, r_cap) == best_oracle.enriched(ss, l, kept, s, r_cap), (round_, s, r_cap)


def test_hash_errors_mirror_the_reference(pm, ctx, example):
    ctx.set_sequences(example.bases, example.offs)
    with pytest.raises(pm.PmError) as e:
        ctx.hash_trial(12, list(range(1, 13)), backend=0)  # test_projection.cpp:243-249
    assert e.value.kind == "DenseTableTooLargeError"
    ctx.hash_trial(12, list(range(1, 13)), backend=2)
    ctx.hash_trial(12, list(range(1, 13)), backend=1)
    for kept in ([], [0, 1], [1, 13], [2, 2]):
        with pytest.raises(pm.PmError) as e:
            ctx.hash_trial(12, kept)
        assert e.value.kind == "InvalidParamsError"
    for s, r in ((0, 5), (3, 2)):
        with pytest.raises(pm.PmError) as e:
            ctx.enriched_buckets(8, [1, 2, 3, 6, 7], s, r)
        assert e.value.kind == "InvalidParamsError"
    with pytest.raises(pm.PmError) as e:
        ctx.hash_keys(41, [1, 2])  # a sequence shorter than l
    assert e.value.kind in ("InvalidParamsError", "Unsupported")


def test_challenge_scale_hashing_matches_reference_goldens(ctx, golden, instance):
    for h in golden["hash"]:
        ss, _, _ = instance(*h["instance"])
        ctx.set_sequences(ss.bases, ss.offs)
        assert sha(ctx.hash_keys(h["l"], h["kept"]).astype("<u8").tobytes()) == h["keys_sha256"]
        bk, bs, bm = ctx.hash_trial(h["l"], h["kept"])
        assert len(bk) == h["n_buckets"]
        assert sha(bk.astype("<u8").tobytes()) == h["bucket_keys_sha256"]
        assert sha(bs.astype("<i4").tobytes()) == h["bucket_sizes_sha256"]
        assert sha(bm.astype("<i4").tobytes()) == h["members_sha256"]
        assert ctx.enriched_buckets(h["l"], h["kept"], h["s"], ss.t * h["s"]) == h["enriched"]


def check_candidate(got, want_consensus, want_positions, want_score, want_iterations, want_expectation, want_theta):
    assert got["consensus"] == want_consensus
    assert got["positions"] == want_positions
    assert got["score"] == want_score
    assert got["iterations"] == want_iterations
    assert abs(got["expectation"] - want_expectation) <= EXPECTATION_TOL
    assert np.abs(got["theta"].astype(np.float64) - np.asarray(want_theta)).max() <= THETA_TOL


def test_refine_matches_reference_goldens(ctx, golden, instance):
    by_inst = {}
    for g in golden["refine"]:
        by_inst.setdefault(tuple(g["instance"]), []).append(g)
    for key, items in by_inst.items():
        ss, _, _ = instance(*key)
        ctx.set_sequences(ss.bases, ss.offs)
        got = ctx.refine(items[0]["l"], [g["members"] for g in items])
        for a, g in zip(got, items):
            check_candidate(a, g["consensus"], g["positions"], g["score"], g["iterations"], g["expectation"], g["theta"])
            np.testing.assert_allclose(a["ll_trace"], g["ll_trace"], atol=1e-3, rtol=0)


def test_refine_worked_example(ctx, example, golden):
    # test_refine.cpp:154-163
    w = golden["worked"]
    ctx.set_sequences(example.bases, example.offs)
    got = ctx.refine(8, [w["enriched_s4"][0]["members"]])[0]
    g = w["refine"]
    check_candidate(got, "ATGCAACT", EXAMPLE_STARTS, 53, g["iterations"], g["expectation"], g["theta"])


def test_refine_matches_oracle_on_random_instances(ctx, best_oracle):
    # small random sets: EM saturates, stops early and window weights tie -- the cases the FP32 kernels hand to the
    # FP64-assisted ones (argmax near-ties: pair kernel; stop decisions near tol: FP64 kernel).  Everything must match.
    rng = np.random.default_rng(15)
    compared = 0
    for round_ in range(12):
        t, l = int(rng.integers(3, 9)), int(rng.integers(3, 14))
        ss = random_set(rng, t, l + 5, l + 70)
        k = max(1, l - 2)
        kept = best_oracle.sample_plan(l, k, round_)
        en = best_oracle.enriched(ss, l, kept, 1, t)[:12]
        ctx.set_sequences(ss.bases, ss.offs)
        for mode in ("2", "0"):  # through the tensor-core kernel and on the pair kernel alone
            os.environ["PM_B200_EM_TC"] = mode
            try:
                got = ctx.refine(l, [e["members"] for e in en])
            finally:
                os.environ.pop("PM_B200_EM_TC", None)
            for e, a in zip(en, got):
                w = best_oracle.refine(ss, l, e["members"], e["key"])
                check_candidate(a, w.consensus, w.positions, w.score, w.iterations, w.expectation, w.theta)
                compared += 1
    assert compared >= 200


def test_stage_exports_init_model_em_step_expectation(pm, ctx, golden, example, instance, best_oracle):
    """pm_init_model / pm_em_step / pm_em_step_exact / pm_expectation against the reference's own stage goldens
    (refine.hpp:90,130,216; test_refine.cpp:28-56, :82-127)."""
    w = golden["worked"]
    ctx.set_sequences(example.bases, example.offs)
    th0 = ctx.init_model(8, w["enriched_s4"][0]["members"])
    np.testing.assert_allclose(th0, np.array(w["theta0"]), atol=1e-15, rtol=0)   # theta0 in sevenths, bit for bit
    assert abs(pm.expectation(th0, 8) - 53.0 / 7) < 1e-12
    np.testing.assert_allclose(th0[:, 0], [76 / 280, 66 / 280, 73 / 280, 65 / 280], atol=1e-15)
    g = golden["em_step"]
    ss, _, _ = instance(*g["instance"])
    ctx.set_sequences(ss.bases, ss.offs)
    th = ctx.init_model(g["l"], g["members"], g["pseudocount"])
    np.testing.assert_allclose(th, np.array(g["theta0"]), atol=1e-15, rtol=0)
    th1x, llx = ctx.em_step(g["l"], th, exact=True)          # FP64 kernel: the reference to rounding
    np.testing.assert_allclose(th1x, np.array(g["theta1"]), atol=1e-12, rtol=0)
    assert abs(llx - g["ll"]) < 1e-9
    th1, ll = ctx.em_step(g["l"], th)                         # production kernel: stated FP32 tolerances
    np.testing.assert_allclose(th1, np.array(g["theta1"]), atol=THETA_TOL, rtol=0)
    assert abs(ll - g["ll"]) < 1e-3
    # column-stochastic after each step, likelihood non-decreasing (test_refine.cpp:101-127), both kernels
    for exact in (False, True):
        model, prev = th, -np.inf
        for _ in range(5):
            model, ll = ctx.em_step(g["l"], model, exact=exact)
            assert np.abs(model.sum(axis=0) - 1.0).max() < (1e-9 if exact else 1e-6)
            assert ll >= prev - (1e-6 if exact else 1e-3)
            want_model, want_ll = best_oracle.em_step(ss, g["l"], model)
            prev = ll
    for bad, kind in (((8, [], 0.0), "EmptyBucketError"), ((8, [1], -0.5), "InvalidParamsError"), ((8, [10 ** 7], 0.0), "IndexOutOfRangeError")):
        with pytest.raises(pm.PmError) as e:
            ctx.init_model(*bad)
        assert e.value.kind == kind


def test_trial_plans_sampled_on_the_device(pm, ctx):
    """pm_run samples seed-derived plans on the device (csrc/pm_plans.cuh: splitmix64 seed, the first outputs of
    mt19937_64 from its seeding chain, uniform_below with rejection, partial Fisher-Yates, sorted complement): the
    same kept positions as the host's pm_trial_plan -- itself pinned to the reference's stream -- for every motif
    length, k = 1 ... l, master seeds including 0 and 2^64-1, strided trials and trial numbers beyond 2^32."""
    rng = np.random.default_rng(99)
    cases = [(15, 7, 7, 1, 172, 1), (20, 7, 7, 1, 3421, 1), (31, 1, 0, 1, 40, 1), (31, 30, 2**64 - 1, 5, 33, 3),
             (1, 1, 5, 1, 4, 1), (8, 8, 11, 2, 9, 1), (19, 6, 123456789, 2**33, 65, 7)]
    for _ in range(12):
        l = int(rng.integers(2, 32))
        cases.append((l, int(rng.integers(1, l + 1)), int(rng.integers(0, 2**63)), int(rng.integers(1, 10**6)),
                      int(rng.integers(1, 300)), int(rng.integers(1, 9))))
    for l, k, seed, first, n, stride in cases:
        got = ctx.trial_plans_device(l, k, seed, first, n, stride)
        for i in (0, 1, n // 2, n - 1):
            assert got[i].tolist() == pm.trial_plan(l, k, seed, first + i * stride), (l, k, seed, first, stride, i)
        if n <= 200:
            assert all(got[i].tolist() == pm.trial_plan(l, k, seed, first + i * stride) for i in range(n))


def test_planted_instances_generated_on_the_device(pm, ctx, golden):
    """pm_ctx_generate_planted (planted.hpp:38-101 on the device): same bytes, motif and positions as the reference for
    every pinned instance, the set is loaded in the context, and a config-5-sized instance equals the host generator."""
    import hashlib
    for p in golden["planted"]:
        bases, offs, motif, pos = ctx.generate_planted(p["t"], p["n"], p["l"], p["d"], p["seed"])
        assert (motif, pos, hashlib.sha256(bases).hexdigest()) == (p["motif"], p["positions"], p["sha256"]), p
        assert ctx.total_lmers(p["l"]) == p["t"] * (p["n"] - p["l"] + 1)
    # the loaded set is what the hashing stage sees
    h = [x for x in golden["hash"] if x["instance"] == [20, 600, 15, 4, 42] and x["trial"] == 1 and x["k"] == 7][0]
    ctx.generate_planted(20, 600, 15, 4, 42)
    assert sha(ctx.hash_keys(15, h["kept"]).astype("<u8").tobytes()) == h["keys_sha256"]
    assert ctx.symbol_counts() == [bytes(pm.generate_planted(20, 600, 15, 4, 42)[0]).count(c) for c in (b"A", b"C", b"T", b"G")]
    want = pm.generate_planted(2000, 1000, 15, 4, 42)
    got = ctx.generate_planted(2000, 1000, 15, 4, 42)
    assert got[0] == want[0] and got[2:] == want[2:]
    n_eq_l = ctx.generate_planted(3, 8, 8, 2, 9)  # n == l: no start draw at all
    assert n_eq_l[0] == pm.generate_planted(3, 8, 8, 2, 9)[0] and n_eq_l[3] == [1, 1, 1]
    for bad in ((0, 10, 3, 1), (2, 10, 11, 1), (2, 10, 3, 3)):
        with pytest.raises(pm.PmError) as e:
            ctx.generate_planted(*bad, 1)
        assert e.value.kind == "InvalidParamsError"


def test_run_multi_equals_single_context(pm, ctx, golden, instance):
    """pm_run_multi over a device list (contexts may share a GPU): contiguous and round-robin shards give the
    single-context result, per-trial bucket counts and early stop included."""
    ss, _, _ = instance(20, 600, 15, 4, 42)
    kw = dict(l=15, d=4, k=7, s=4, m=16, seed=7, early_stop=0)
    want = [r for r in golden["run"] if r["cfg"].get("m") == 16][0]["result"]
    for devices in ([0], [0, 0], [0, 0, 0], [0] * 5):
        for strided in (False, True):
            r = pm.run_multi(devices, ss.bases, ss.offs, strided=strided, **kw)
            for f in ("consensus", "score", "iterations", "source_bucket", "best_trial", "trials_run", "buckets_enriched", "positions"):
                assert r[f] == want[f], (devices, strided, f, r[f], want[f])
            assert abs(r["expectation"] - want["expectation"]) <= EXPECTATION_TOL
    # early stop: a d = 0 plant is perfect at trial 1 whichever shard holds it
    ss, motif, _ = instance(5, 50, 10, 0, 77)
    ctx.set_sequences(ss.bases, ss.offs)
    one = ctx.run(l=10, d=0, seed=5, m=10)
    for devices in ([0, 0], [0, 0, 0]):
        for strided in (False, True):
            r = pm.run_multi(devices, ss.bases, ss.offs, strided=strided, l=10, d=0, seed=5, m=10)
            assert (r["consensus"], r["score"], r["best_trial"], r["trials_run"], r["buckets_enriched"]) == \
                   (motif, 50, one["best_trial"], one["trials_run"], one["buckets_enriched"])
    with pytest.raises(pm.PmError) as e:
        pm.run_multi([0, 0], ss.bases, ss.offs, l=10, d=12)
    assert e.value.kind == "InvalidParamsError"


def test_refine_single_member_and_limits(pm, ctx, best_oracle, instance):
    ss, _, pos = instance(6, 30, 5, 0, 99)
    ctx.set_sequences(ss.bases, ss.offs)
    # exact plant recovered with a perfect score (test_refine.cpp:165-175)
    members = [ss.ref_to_flat(5, i + 1, pos[i]) for i in range(6)]
    got = ctx.refine(5, [members])[0]
    want = best_oracle.refine(ss, 5, members)
    assert (got["consensus"], got["score"], got["positions"]) == (want.consensus, 30, pos)
    # max_iters = 1 and a looser tolerance are honoured
    for iters, tol in ((1, 1e-6), (3, 1e-6), (5, 10.0)):
        a = ctx.refine(5, [members[:2]], max_iters=iters, tol=tol)[0]
        b = best_oracle.refine(ss, 5, members[:2], max_iters=iters, tol=tol)
        assert a["iterations"] == b.iterations and a["positions"] == b.positions
    with pytest.raises(pm.PmError) as e:
        ctx.refine(5, [members], max_iters=0)
    assert e.value.kind == "InvalidParamsError"
    with pytest.raises(pm.PmError) as e:
        ctx.refine(5, [[]])
    assert e.value.kind == "EmptyBucketError"
    with pytest.raises(pm.PmError) as e:
        ctx.refine(5, [[10 ** 6]])
    assert e.value.kind == "IndexOutOfRangeError"


def test_m_step_cutoff_is_within_its_bound(ctx, golden, instance):
    """z_epsilon=0 adds every window's responsibility (the reference's dense M-step); the default
    cut-off 2^-30 may drop at most W*eps of mass per count."""
    g = [x for x in golden["refine"] if x["instance"][1] == 600][:8]
    ss, _, _ = instance(*g[0]["instance"])
    ctx.set_sequences(ss.bases, ss.offs)
    dense = ctx.refine(15, [x["members"] for x in g], z_epsilon=0.0)
    sparse = ctx.refine(15, [x["members"] for x in g])
    for a, b, x in zip(dense, sparse, g):
        assert np.abs(a["theta"] - b["theta"]).max() <= 586 * 2.0 ** -30 + 1e-6
        assert (a["positions"], a["score"], a["consensus"]) == (b["positions"], b["score"], b["consensus"])
        check_candidate(a, x["consensus"], x["positions"], x["score"], x["iterations"], x["expectation"], x["theta"])


def test_score_and_hamming_scan_match_oracle(ctx, best_oracle):
    rng = np.random.default_rng(5)
    for _ in range(10):
        l = int(rng.integers(1, 32))
        ss = random_set(rng, int(rng.integers(1, 8)), l, l + 80)
        ctx.set_sequences(ss.bases, ss.offs)
        starts = [int(rng.integers(1, int(ss.offs[i + 1] - ss.offs[i]) - l + 2)) for i in range(ss.t)]
        assert ctx.score(l, starts) == best_oracle.score(ss, l, starts)
        v = "".join(rng.choice(list("ACGT"), l))
        per, tot, within = ctx.hamming_scan(v, 2)
        wtot, wper = best_oracle.total_distance(ss, v)
        assert (tot, per) == (wtot, wper) and within == sum(1 for p in wper if p <= 2)
    # consensus ties: A over C, T over G (test_scoring.cpp:81-91)
    ss = pmo.SeqSet.from_strings(["AT", "CG"])
    ctx.set_sequences(ss.bases, ss.offs)
    assert ctx.score(2, [1, 1]) == (2, "AT")


def test_tiled_em_equals_single_tile_and_reference(pm, golden, instance):
    """Large sets are swept in sequence tiles; forcing small tiles on a golden
    instance must reproduce the reference candidates exactly like the single-tile layout."""
    import os
    g = [x for x in golden["refine"] if x["instance"][1] == 600][:10]
    ss, _, _ = instance(*g[0]["instance"])
    results = {}
    for slots in (None, 4000, 1500):
        if slots is None:
            os.environ.pop("PM_B200_TILE_SLOTS", None)
        else:
            os.environ["PM_B200_TILE_SLOTS"] = str(slots)
        try:
            with pm.Context(0) as c:
                c.set_sequences(ss.bases, ss.offs)
                results[slots] = c.refine(15, [x["members"] for x in g])
        finally:
            os.environ.pop("PM_B200_TILE_SLOTS", None)
    for slots, res in results.items():
        for a, x in zip(res, g):
            check_candidate(a, x["consensus"], x["positions"], x["score"], x["iterations"], x["expectation"], x["theta"])
    for a, b in zip(results[None], results[1500]):
        assert np.abs(a["theta"] - b["theta"]).max() < 1e-6


def test_many_sequences_multi_tile_matches_oracle(ctx, best_oracle):
    """t = 300 ragged sequences (about 60k bases => several tiles, previous maxima in global memory
    is exercised separately by t > 1024 in test_gpu_run)."""
    rng = np.random.default_rng(99)
    ss = random_set(rng, 300, 150, 250)
    l, kept = 11, [1, 2, 4, 5, 7, 8, 10, 11]
    ctx.set_sequences(ss.bases, ss.offs)
    en = best_oracle.enriched(ss, l, kept, 5, 300 * 5)
    assert ctx.enriched_buckets(l, kept, 5, 300 * 5) == en
    pick = en[:6]
    got = ctx.refine(l, [e["members"] for e in pick])
    for e, a in zip(pick, got):
        w = best_oracle.refine(ss, l, e["members"], e["key"])
        check_candidate(a, w.consensus, w.positions, w.score, w.iterations, w.expectation, w.theta)


def test_streaming_fallback_kernel_matches_reference(pm, golden, instance):
    """A sequence longer than a tile cannot use the shared-memory EM kernel; the streaming kernel
     takes over.  Forced here by a tile budget smaller than one sequence."""
    import os
    g = [x for x in golden["refine"] if x["instance"][1] == 600][:6]
    ss, _, _ = instance(*g[0]["instance"])
    os.environ["PM_B200_TILE_SLOTS"] = "300"
    try:
        with pm.Context(0) as c:
            c.set_sequences(ss.bases, ss.offs)
            res = c.refine(15, [x["members"] for x in g])
            dense = c.refine(15, [x["members"] for x in g[:2]], z_epsilon=0.0)
            run = c.run(l=15, d=4, k=7, s=4, m=2, seed=7, early_stop=0)
    finally:
        os.environ.pop("PM_B200_TILE_SLOTS", None)
    for a, x in zip(res, g):
        check_candidate(a, x["consensus"], x["positions"], x["score"], x["iterations"], x["expectation"], x["theta"])
    for a, b in zip(dense, res):
        assert np.abs(a["theta"] - b["theta"]).max() <= 586 * 2.0 ** -30 + 1e-6
    want = [r for r in golden["run"] if r["cfg"].get("m") == 16][0]["result"]
    assert run["score"] <= want["score"] and run["buckets_enriched"] == sum(golden["trial_outcomes_c1"]["buckets"][:2])
