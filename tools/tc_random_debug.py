"""Debug helper: the randomized tensor-core parity cases of tests/test_gpu_em_pair.py, per kernel tier."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1605_06904_b200 as pm  # noqa: E402
from oracle import pmo  # noqa: E402

oracle = pmo.load("reference" if pmo.available("reference") else "port")
rng = np.random.default_rng(1605)
for l, t, iters in ((5, 7, 5), (8, 2, 3), (11, 13, 5), (12, 40, 2), (13, 9, 8), (16, 21, 1), (17, 5, 5), (20, 30, 4)):
    ss = pmo.SeqSet.from_strings(["".join(rng.choice(list("ACGT"), int(rng.integers(l + 30, 420)))) for _ in range(t)])
    kept = oracle.sample_plan(l, min(l - 1, 6), 100 + l)
    en = oracle.enriched(ss, l, kept, 1, 4 * t)
    en = en[:: max(1, len(en) // 150)][:150]
    want = [oracle.refine(ss, l, e["members"], e["key"], max_iters=iters) for e in en]
    for mode in ("2", "0", "exact"):
        if mode != "exact":
            os.environ["PM_B200_EM_TC"] = mode
        with pm.Context(0) as c:
            c.set_sequences(ss.bases, ss.offs)
            got = c.refine(l, [e["members"] for e in en], max_iters=iters, exact=(mode == "exact"))
            counts = c.em_exact_counts()
        bad = 0
        for b, (a, w) in enumerate(zip(got, want)):
            if (a["consensus"], a["score"], a["positions"], a["iterations"]) != (w.consensus, w.score, w.positions, w.iterations):
                bad += 1
                if bad <= 2:
                    diff = [i for i in range(t) if a["positions"][i] != w.positions[i]]
                    print(f"   l={l} t={t} iters={iters} mode={mode} bucket {b} members {len(en[b]['members'])}: score {a['score']}/{w.score} "
                          f"iters {a['iterations']}/{w.iterations} positions differ at {diff[:6]} got {[a['positions'][i] for i in diff[:6]]} "
                          f"want {[w.positions[i] for i in diff[:6]]} dE {a['expectation'] - w.expectation:.3g}")
        print(f"l={l} t={t} iters={iters} mode={mode}: {bad}/{len(en)} mismatches, handed over {counts}")
