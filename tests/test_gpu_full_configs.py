"""Parity on every BASELINE.json challenge configuration at FULL size against known answers from the UNMODIFIED
reference (tests/golden/reference_full_<cfg>.json, written by tests/golden/make_full_golden.py from oracle/_ref):

  c1 (15,4) t=20 n=600 m=172 | c2 (16,5) n=1000 m=1293 | c3 (18,6) m=2218 | c3b (19,6) m=711 | c4 (20,7) m=3421

For each: the instance pin, hashing/grouping SHA-256s and the enriched list of trials 1 and m, >= 56 refined buckets
(discrete outputs exact, theta/expectation/likelihood within the stated FP32 tolerances), the outcome of EVERY trial
(enriched count, best score, best bucket key exact; best expectation within tolerance) and the full-m run() result."""
import hashlib
import json
import os

import numpy as np
import pytest

from conftest import EXPECTATION_TOL, REPO, THETA_TOL

pytestmark = pytest.mark.gpu

CONFIGS = ["c1", "c2", "c3", "c3b", "c4"]
LL_TOL = 1e-3  # log-likelihood trace, absolute (|LL| ~ 1.6e4 .. 2.8e4)


def load(name):
    path = os.path.join(REPO, "tests", "golden", f"reference_full_{name}.json")
    if not os.path.exists(path):
        pytest.fail(f"{path} is missing: run tests/golden/make_full_golden.py {name} in the build container")
    with open(path) as f:
        return json.load(f)


def sha(a):
    return hashlib.sha256(a).hexdigest()


@pytest.fixture(scope="module", params=CONFIGS)
def cfg(request, pm, ctx):
    g = load(request.param)
    t, n, l, d, seed = g["instance"]
    bases, offs, motif, pos = pm.generate_planted(t, n, l, d, seed)
    assert sha(bases) == g["sha256"], "generate_planted diverged from the reference instance"
    assert motif == g["motif"] and pos == g["planted_positions"]
    ctx.set_sequences(bases, offs)
    return g


def test_hashing_and_enrichment(cfg, pm, ctx):
    t, n, l, d, _ = cfg["instance"]
    for h in cfg["hash"]:
        kept = pm.trial_plan(l, cfg["k"], cfg["seed"], h["trial"])
        assert kept == h["kept"]
        keys = ctx.hash_keys(l, kept)
        assert sha(keys.astype("<u8").tobytes()) == h["keys_sha256"]
        bk, bs, bm = ctx.hash_trial(l, kept)
        assert len(bk) == h["n_buckets"]
        assert sha(bk.astype("<u8").tobytes()) == h["bucket_keys_sha256"]
        assert sha(bs.astype("<i4").tobytes()) == h["bucket_sizes_sha256"]
        assert sha(bm.astype("<i4").tobytes()) == h["members_sha256"]
        en = ctx.enriched_buckets(l, kept, cfg["s"], t * cfg["s"])
        assert len(en) == h["n_enriched"]
        if h["enriched"] is not None:
            assert en == h["enriched"]


def check_refined(got, want, l):
    for f in ("consensus", "positions", "score", "iterations"):
        assert got[f] == want[f], (f, want["key"], got[f], want[f])
    assert abs(got["expectation"] - want["expectation"]) <= EXPECTATION_TOL
    np.testing.assert_allclose(got["theta"], np.array(want["theta"]), atol=THETA_TOL, rtol=0)
    np.testing.assert_allclose(got["ll_trace"], want["ll_trace"], atol=LL_TOL, rtol=0)


def test_refined_buckets(cfg, ctx):
    l = cfg["instance"][2]
    gold = cfg["refine"]
    assert len(gold) >= 50
    got = ctx.refine(l, [g["members"] for g in gold])
    for a, g in zip(got, gold):
        check_refined(a, g, l)
    # the same buckets through the exact FP64 kernel: the reference's numbers to ~1e-10
    exact = ctx.refine(l, [g["members"] for g in gold[:8]], exact=True)
    for a, g in zip(exact, gold[:8]):
        for f in ("consensus", "positions", "score", "iterations"):
            assert a[f] == g[f]
        assert abs(a["expectation"] - g["expectation"]) <= 1e-9
        np.testing.assert_allclose(a["theta"], np.array(g["theta"]), atol=1e-10, rtol=0)
        np.testing.assert_allclose(a["ll_trace"], g["ll_trace"], atol=1e-7, rtol=0)


def test_every_trial_and_the_full_run(cfg, ctx):
    t, n, l, d, _ = cfg["instance"]
    r = ctx.run(per_trial=True, l=l, d=d, k=cfg["k"], s=cfg["s"], m=cfg["m"], seed=cfg["seed"], early_stop=0)
    o = cfg["outcomes"]
    assert r["trial_buckets"].tolist() == o["buckets"]
    assert r["trial_score"].tolist() == o["score"]
    assert [int(v) for v in r["trial_key"]] == o["key"]
    np.testing.assert_allclose(r["trial_expectation"], o["expectation"], atol=EXPECTATION_TOL, rtol=0)
    want = cfg["run"]
    for f in ("consensus", "score", "iterations", "source_bucket", "best_trial", "trials_run", "buckets_enriched", "k", "s", "m",
              "positions"):
        assert r[f] == want[f], (f, r[f], want[f])
    assert abs(r["expectation"] - want["expectation"]) <= EXPECTATION_TOL
    # where the reference recovers the planted motif (it does not on every challenge instance: a spurious motif can
    # out-score the plant), every sequence holds it within d mismatches
    if want["consensus"] == cfg["motif"]:
        assert r["within_d"] == t


def test_full_run_is_identical_with_the_pair_kernel_only(cfg, ctx):
    """PM_B200_EM_TC=0 keeps every bucket on the exact (FP64-assisted) pair kernel: same run() result."""
    if cfg["config"] not in ("c1", "c3b"):
        pytest.skip("covered on c1 and c3b (the pair kernel alone needs seconds on the larger configurations)")
    t, n, l, d, _ = cfg["instance"]
    os.environ["PM_B200_EM_TC"] = "0"
    try:
        r = ctx.run(l=l, d=d, k=cfg["k"], s=cfg["s"], m=cfg["m"], seed=cfg["seed"], early_stop=0)
    finally:
        os.environ.pop("PM_B200_EM_TC", None)
    want = cfg["run"]
    for f in ("consensus", "score", "iterations", "source_bucket", "best_trial", "buckets_enriched", "positions"):
        assert r[f] == want[f], (f, r[f], want[f])
    assert ctx.em_exact_counts()["total"] == 0
