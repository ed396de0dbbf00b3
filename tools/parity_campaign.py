"""Randomized parity campaign (run on the GPU box): run() and refine() against the unmodified reference on random
sets for a time budget, through every EM tier.  Prints one line per mismatch and a summary.

    python tools/parity_campaign.py [seconds] [seed]
"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1605_06904_b200 as pm  # noqa: E402
from oracle import pmo  # noqa: E402

INT_FIELDS = ("consensus", "score", "iterations", "source_bucket", "best_trial", "trials_run", "buckets_enriched", "positions")


def main():
    budget = float(sys.argv[1]) if len(sys.argv) > 1 else 120.0
    seed = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    oracle = pmo.load("reference" if pmo.available("reference") else "port")
    rng = np.random.default_rng(seed)
    t0 = time.time()
    runs = run_bad = buckets = bucket_bad = 0
    max_dth = max_de = 0.0
    while time.time() - t0 < budget:
        t = int(rng.integers(2, 41))
        l = int(rng.integers(5, 21))
        alphabet = list("ACGT")
        probs = rng.dirichlet(np.ones(4) * rng.choice([0.3, 1.0, 5.0]))  # from skewed to uniform composition
        strings = ["".join(rng.choice(alphabet, int(rng.integers(l + 5, 700)), p=probs)) for _ in range(t)]
        ss = pmo.SeqSet.from_strings(strings)
        k = int(rng.integers(max(1, l - 8), l))
        kw = dict(l=l, d=int(rng.integers(0, 3)), k=k, s=int(rng.integers(1, 5)), m=int(rng.integers(1, 6)),
                  seed=int(rng.integers(0, 2**31)), early_stop=int(rng.integers(0, 2)), max_em_iters=int(rng.integers(1, 8)))
        try:
            want = oracle.run(ss, **kw)
        except Exception as e:  # the reference rejects the parameters: so must we
            want = type(e).__name__
        for mode in ("2", "1", "0"):
            os.environ["PM_B200_EM_TC"] = mode
            with pm.Context(0) as c:
                c.set_sequences(ss.bases, ss.offs)
                try:
                    got = c.run(**kw)
                except pm.PmError as e:
                    got = e.kind
            runs += 1
            if isinstance(want, str) or isinstance(got, str):
                if not (isinstance(want, str) and isinstance(got, str)):
                    run_bad += 1
                    print("RUN MISMATCH (error vs result)", mode, kw, t, want if isinstance(want, str) else "result", got if isinstance(got, str) else "result")
                continue
            bad = [f for f in INT_FIELDS if got[f] != want[f]]
            if bad or abs(got["expectation"] - want["expectation"]) > 1e-3:
                run_bad += 1
                print("RUN MISMATCH", mode, kw, "t", t, bad, [(got[f], want[f]) for f in bad if f != "positions"])
        # refine(): a sample of this set's buckets, tensor-core kernel forced on
        os.environ["PM_B200_EM_TC"] = "2"
        kept = oracle.sample_plan(l, k, int(rng.integers(0, 2**31)))
        en = oracle.enriched(ss, l, kept, 1, 4 * t)
        en = en[:: max(1, len(en) // 60)][:60]
        if en:
            iters = kw["max_em_iters"]
            with pm.Context(0) as c:
                c.set_sequences(ss.bases, ss.offs)
                got = c.refine(l, [e["members"] for e in en], max_iters=iters)
            for e, a in zip(en, got):
                w = oracle.refine(ss, l, e["members"], e["key"], max_iters=iters)
                buckets += 1
                max_dth = max(max_dth, float(np.abs(a["theta"].astype(np.float64) - w.theta).max()))
                max_de = max(max_de, abs(a["expectation"] - w.expectation))
                if (a["consensus"], a["score"], a["positions"], a["iterations"]) != (w.consensus, w.score, w.positions, w.iterations):
                    bucket_bad += 1
                    print("BUCKET MISMATCH", dict(l=l, t=t, iters=iters, members=len(e["members"])),
                          [i for i in range(t) if a["positions"][i] != w.positions[i]][:5], a["iterations"], w.iterations)
    os.environ.pop("PM_B200_EM_TC", None)
    print(f"campaign seed {seed}: {runs} runs ({run_bad} mismatches), {buckets} refined buckets ({bucket_bad} mismatches), "
          f"max|dtheta| {max_dth:.3g}, max|dE| {max_de:.3g}, {time.time() - t0:.0f} s, oracle = {oracle.impl}")


if __name__ == "__main__":
    main()
