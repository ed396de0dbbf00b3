"""The two-buckets-per-CTA EM kernel (csrc/pm_em_pair.cuh): buckets of a pair run in lockstep, so the
cases that matter are the ones where the two differ -- one converges early and is frozen while the other
keeps iterating, an odd tail, a different partner -- and agreement with the one-bucket kernel."""
import os

import numpy as np
import pytest

from conftest import EXPECTATION_TOL, THETA_TOL

pytestmark = pytest.mark.gpu


def _check(a, w):
    assert a["iterations"] == w.iterations
    assert a["positions"] == w.positions
    assert (a["consensus"], a["score"]) == (w.consensus, w.score)
    assert abs(a["expectation"] - w.expectation) <= EXPECTATION_TOL
    assert np.abs(a["theta"].astype(np.float64) - w.theta).max() <= THETA_TOL


def test_pairs_with_different_iteration_counts(ctx, best_oracle, instance):
    """refine.hpp:296-304 stops each bucket on its own likelihood gain; with max_iters = 12 the enriched
    buckets of this easy instance stop after 3..12 iterations, so most pairs hold a frozen bucket."""
    t, n, l, d, seed = 10, 80, 7, 0, 11
    ss, _, _ = instance(t, n, l, d, seed)
    kept = best_oracle.sample_plan(l, 5, 1)
    en = best_oracle.enriched(ss, l, kept, 2, t * 2)[:41]  # odd count: the last CTA refines a lone bucket
    want = [best_oracle.refine(ss, l, e["members"], e["key"], max_iters=12) for e in en]
    its = [w.iterations for w in want]
    assert len(set(its)) >= 4 and any(its[i] != its[i + 1] for i in range(0, 40, 2)), its
    ctx.set_sequences(ss.bases, ss.offs)
    got = ctx.refine(l, [e["members"] for e in en], max_iters=12)
    for a, w in zip(got, want):
        _check(a, w)
        np.testing.assert_allclose(a["ll_trace"][: w.iterations], w.ll_trace, atol=5e-2, rtol=0)


def test_result_does_not_depend_on_the_partner(ctx, best_oracle, instance):
    """A bucket's outputs are a function of the bucket alone: any pairing gives bit-identical results."""
    ss, _, _ = instance(12, 120, 8, 0, 5)
    kept = best_oracle.sample_plan(8, 5, 1)
    en = best_oracle.enriched(ss, 8, kept, 2, 24)[:9]
    ctx.set_sequences(ss.bases, ss.offs)
    members = [e["members"] for e in en]
    base = ctx.refine(8, members)
    order = [4, 0, 8, 2, 6, 1, 7, 3, 5]
    shuffled = ctx.refine(8, [members[i] for i in order])
    alone = [ctx.refine(8, [m])[0] for m in members[:3]]
    for pos, i in enumerate(order):
        a, b = base[i], shuffled[pos]
        assert (a["consensus"], a["score"], a["positions"], a["iterations"]) == \
               (b["consensus"], b["score"], b["positions"], b["iterations"])
        assert a["expectation"] == b["expectation"] and (a["theta"] == b["theta"]).all()
    for a, b in zip(base, alone):
        assert a["expectation"] == b["expectation"] and (a["theta"] == b["theta"]).all()


def test_tensor_core_kernel_agrees_with_pair_kernel(pm, golden, instance):
    """PM_B200_EM_TC=0 keeps every bucket on the pair kernel, 2 sends even a handful through the tensor-core kernel
    (pm_em_tc.cuh): same discrete outputs on the challenge-scale goldens, thetas within FP32 noise of each other."""
    g = [x for x in golden["refine"] if x["instance"][1] == 600][:7]
    ss, _, _ = instance(*g[0]["instance"])
    res = {}
    for flag in ("2", "0"):
        os.environ["PM_B200_EM_TC"] = flag
        try:
            with pm.Context(0) as c:
                c.set_sequences(ss.bases, ss.offs)
                res[flag] = c.refine(15, [x["members"] for x in g])
                exact = c.em_exact_counts()["total"]
                assert exact == 0 if flag == "0" else exact <= len(g)
        finally:
            os.environ.pop("PM_B200_EM_TC", None)
    for a, b, x in zip(res["2"], res["0"], g):
        assert (a["consensus"], a["score"], a["positions"], a["iterations"]) == \
               (b["consensus"], b["score"], b["positions"], b["iterations"]) == \
               (x["consensus"], x["score"], x["positions"], x["iterations"])
        assert np.abs(a["theta"] - b["theta"]).max() < 2e-5
        assert abs(a["expectation"] - x["expectation"]) <= EXPECTATION_TOL


def test_tensor_core_kernel_on_random_shapes(pm, best_oracle):
    """The tensor-core kernel forced on (PM_B200_EM_TC=2) across its four operand widths (l = 5 ... 20 -> K = 32, 48,
    64, 80), ragged sequence lengths (segments that end in the middle of a chunk, blocks of every size), 2 ... 40
    sequences and iteration budgets 1 ... 8, against the reference: discrete outputs strictly equal -- whatever the
    kernel cannot decide with margin it hands to the exact kernels -- and theta / expectation within tolerance.  The
    exponent range of its single per-bucket reference (64 ... 108 binades under the weight bound) is exercised by theta0's
    floored columns: buckets of one or two members."""
    from oracle import pmo
    rng = np.random.default_rng(1605)
    os.environ["PM_B200_EM_TC"] = "2"
    try:
        total = handed = 0
        for l, t, iters in ((5, 7, 5), (8, 2, 3), (11, 13, 5), (12, 40, 2), (13, 9, 8), (16, 21, 1), (17, 5, 5), (20, 30, 4)):
            ss = pmo.SeqSet.from_strings(["".join(rng.choice(list("ACGT"), int(rng.integers(l + 30, 420)))) for _ in range(t)])
            kept = best_oracle.sample_plan(l, min(l - 1, 6), 100 + l)
            en = best_oracle.enriched(ss, l, kept, 1, 4 * t)
            en = en[:: max(1, len(en) // 150)][:150]
            with pm.Context(0) as c:
                c.set_sequences(ss.bases, ss.offs)
                got = c.refine(l, [e["members"] for e in en], max_iters=iters)
                handed += c.em_exact_counts()["total"]
            for e, a in zip(en, got):
                w = best_oracle.refine(ss, l, e["members"], e["key"], max_iters=iters)
                assert (a["consensus"], a["score"], a["positions"], a["iterations"]) == (w.consensus, w.score, w.positions, w.iterations), (l, t, iters)
                assert np.abs(a["theta"].astype(np.float64) - w.theta).max() <= THETA_TOL
                assert abs(a["expectation"] - w.expectation) <= EXPECTATION_TOL
            total += len(en)
        # buckets of one member put most columns of theta0 at the floor: many of them leave the exponent range of the
        # kernel's single reference (64 binades under the bound for l <= 16) and are handed over -- not all of them
        assert total > 800 and handed < 3 * total // 4
    finally:
        os.environ.pop("PM_B200_EM_TC", None)


def test_long_motifs_use_the_wide_flush_path(ctx, best_oracle):
    """l > 16 means more than eight column pairs: 32-value class flushes, l = 31 fills the whole 64-bit window."""
    import numpy as np
    from oracle import pmo
    rng = np.random.default_rng(77)
    compared = 0
    for l in (17, 20, 24, 31):
        t = 6
        ss = pmo.SeqSet.from_strings(["".join(rng.choice(list("ACGT"), int(rng.integers(l + 20, l + 120)))) for _ in range(t)])
        k = min(l - 2, 12)
        kept = best_oracle.sample_plan(l, k, l)
        en = best_oracle.enriched(ss, l, kept, 1, t)[:7]
        ctx.set_sequences(ss.bases, ss.offs)
        got = ctx.refine(l, [e["members"] for e in en])
        for e, a in zip(en, got):
            w = best_oracle.refine(ss, l, e["members"], e["key"])
            assert a["iterations"] == w.iterations
            assert np.abs(a["theta"].astype(np.float64) - w.theta).max() <= THETA_TOL
            assert abs(a["expectation"] - w.expectation) <= EXPECTATION_TOL
            if a["positions"] == w.positions:
                assert (a["consensus"], a["score"]) == (w.consensus, w.score)
                compared += 1
    assert compared >= 20


def test_large_set_path_with_frozen_buckets(ctx, best_oracle):
    """t > 64 selects the pair kernel's large-set path (per-tile metadata, previous maxima in global memory,
    double-buffered word stages); with max_iters = 12 the buckets of a pair stop at different iterations."""
    import numpy as np
    from oracle import pmo
    rng = np.random.default_rng(5)
    motif = "ACGTTGCA"
    strings = []
    for _ in range(90):
        s = list(rng.choice(list("ACGT"), int(rng.integers(40, 90))))
        at = int(rng.integers(0, len(s) - 8))
        s[at:at + 8] = list(motif)
        strings.append("".join(s))
    ss = pmo.SeqSet.from_strings(strings)
    kept = best_oracle.sample_plan(8, 6, 2)
    en = best_oracle.enriched(ss, 8, kept, 3, 90 * 3)[:15]
    want = [best_oracle.refine(ss, 8, e["members"], e["key"], max_iters=12) for e in en]
    assert len({w.iterations for w in want}) >= 2
    ctx.set_sequences(ss.bases, ss.offs)
    got = ctx.refine(8, [e["members"] for e in en], max_iters=12)
    for a, w in zip(got, want):
        _check(a, w)


def test_near_ties_behind_repeats_of_the_winning_lmer(pm, best_oracle):
    """tests/golden/near_tie_cases.json: buckets of random two-sequence sets on which the reference's argmax
    (refine.hpp:311-316) chooses between two DIFFERENT l-mers whose FP64 weights differ by 1e-10 .. 9e-8 -- in three of
    them the winning l-mer also occurs two or three times in the sequence (bit-identical weights), which used to hide the
    other l-mer from the near-tie test.  Every tier must hand these to the FP64 kernel and return the reference's
    positions; the fixture's `want` is re-checked against the oracle."""
    import json
    from oracle import pmo
    path = os.path.join(os.path.dirname(__file__), "golden", "near_tie_cases.json")
    cases = json.load(open(path))["cases"]
    assert len(cases) == 6
    for cs in cases:
        ss = pmo.SeqSet.from_strings(cs["strings"])
        w = best_oracle.refine(ss, cs["l"], cs["members"], 0, max_iters=cs["max_iters"])
        if best_oracle.impl == "reference":  # gaps of 1e-10 in a window weight: only the reference itself is the judge
            assert (w.consensus, w.score, list(w.positions), w.iterations) == \
                   (cs["want"]["consensus"], cs["want"]["score"], cs["want"]["positions"], cs["want"]["iterations"])
        for mode in ("2", "1", "0"):
            os.environ["PM_B200_EM_TC"] = mode
            try:
                with pm.Context(0) as c:
                    c.set_sequences(ss.bases, ss.offs)
                    a = c.refine(cs["l"], [cs["members"]], max_iters=cs["max_iters"])[0]
                    assert c.em_exact_counts()["fp64"] == 1, (mode, cs["origin"])
            finally:
                os.environ.pop("PM_B200_EM_TC", None)
            assert (a["consensus"], a["score"], list(a["positions"]), a["iterations"]) == \
                   (cs["want"]["consensus"], cs["want"]["score"], cs["want"]["positions"], cs["want"]["iterations"]), (mode, cs["origin"])
            assert abs(a["expectation"] - cs["want"]["expectation"]) <= EXPECTATION_TOL


def test_run_decided_by_the_last_bit_of_saturated_expectations(pm, best_oracle):
    """tests/golden/near_tie_cases.json `runs`: every trial's best bucket is a saturated model (each column one symbol,
    the rest on the 1e-9 floor), so the expectations are 6 / (1 + 3e-9) up to the rounding of the M-step sums, and
    candidate_improves (driver.hpp:127-135) compares them exactly: the reference's winner is trial 1 because trial 2's
    expectation is one ulp smaller.  The FP64 kernel adds every observable sum in the reference's order
    (csrc/pm_em_f64.cuh), so the per-trial expectations are bit-identical and so is the winner, through every tier."""
    import json
    from oracle import pmo
    path = os.path.join(os.path.dirname(__file__), "golden", "near_tie_cases.json")
    for cs in json.load(open(path))["runs"]:
        ss = pmo.SeqSet.from_strings(cs["strings"])
        if best_oracle.impl == "reference":  # the fixture is the reference's output to the last bit; the C port is not held to that
            want = best_oracle.run(ss, **cs["kw"])
            for f, v in cs["want"].items():
                assert (want[f].tolist() if hasattr(want[f], "tolist") else want[f]) == v, f
        for mode in ("2", "1", "0"):
            os.environ["PM_B200_EM_TC"] = mode
            try:
                with pm.Context(0) as c:
                    c.set_sequences(ss.bases, ss.offs)
                    got = c.run(per_trial=True, **cs["kw"])
            finally:
                os.environ.pop("PM_B200_EM_TC", None)
            for f, v in cs["want"].items():
                assert got[f] == v, (mode, f, got[f], v)  # the expectation too: exact
            assert got["trial_buckets"].tolist() == cs["trial_buckets"]
            assert got["trial_score"].tolist() == cs["trial_score"]
            assert got["trial_key"].tolist() == cs["trial_key"]
            # a trial's own record is the FP64 kernel's only where it had to be settled; the winner's always is
            np.testing.assert_allclose(got["trial_expectation"], cs["trial_expectation"], atol=EXPECTATION_TOL, rtol=0)
