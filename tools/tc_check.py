"""Tensor-core EM kernel against the pair kernel on the same buckets (run on the GPU box):
    python tools/tc_check.py [c1|c2|c3|c3b|c4] [trials]
Discrete outputs must be identical; theta / expectation / LL differences and the number of buckets handed to the
exact kernel are printed.  Then pm_run is timed with either kernel."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1605_06904_b200 as pm  # noqa: E402

CFG = {"c1": (20, 600, 15, 4, 172), "c2": (20, 1000, 16, 5, 1293), "c3": (20, 1000, 18, 6, 2218),
       "c3b": (20, 1000, 19, 6, 711), "c4": (20, 1000, 20, 7, 3421)}


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c1"
    ntr = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    t, n, l, d, m = CFG[name]
    bases, offs, motif, _ = pm.generate_planted(t, n, l, d, 42)
    with pm.Context(0) as ctx:
        ctx.set_sequences(bases, offs)
        lists = []
        for tr in range(1, ntr + 1):
            kept = pm.trial_plan(l, 7, 7, tr)
            lists += [e["members"] for e in ctx.enriched_buckets(l, kept, 4, t * 4)]
        print(f"{name}: {len(lists)} buckets from {ntr} trials")
        os.environ["PM_B200_EM_TC"] = "0"
        ref = ctx.refine(l, lists)
        os.environ["PM_B200_EM_TC"] = "2"
        t0 = time.time()
        got = ctx.refine(l, lists)
        print("tc refine wall", time.time() - t0, "exact-kernel buckets:", ctx.em_exact_counts())
        bad = 0
        dth = dex = dll = 0.0
        for b, (a, g) in enumerate(zip(ref, got)):
            same = (a["positions"] == g["positions"] and a["score"] == g["score"] and a["consensus"] == g["consensus"]
                    and a["iterations"] == g["iterations"])
            if not same:
                bad += 1
                if bad <= 5:
                    print("MISMATCH bucket", b, a["score"], g["score"], a["iterations"], g["iterations"], a["consensus"], g["consensus"],
                          [i for i in range(t) if a["positions"][i] != g["positions"][i]])
            dth = max(dth, float(np.abs(a["theta"] - g["theta"]).max()))
            dex = max(dex, abs(a["expectation"] - g["expectation"]))
            if len(a["ll_trace"]) == len(g["ll_trace"]) and a["ll_trace"]:
                dll = max(dll, float(np.abs(np.array(a["ll_trace"]) - np.array(g["ll_trace"])).max()))
        print(f"discrete mismatches {bad}/{len(lists)}  max|dtheta| {dth:.3g}  max|dE| {dex:.3g}  max|dLL| {dll:.3g}")

        for mode in ("0", "1"):
            os.environ["PM_B200_EM_TC"] = mode
            kw = dict(l=l, d=d, k=7, s=4, m=min(m, 400), seed=7, early_stop=0, profile=1)
            r = ctx.run(**kw)
            ts = []
            for _ in range(3):
                t0 = time.time()
                r = ctx.run(**kw)
                ts.append(time.time() - t0)
            print(f"EM_TC={mode}: run m={kw['m']} best {min(ts) * 1e3:.2f} ms  em stage {r['stage_ms'][3]:.2f} ms  -> {r['consensus']} {r['score']} "
                  f"E={r['expectation']:.9f} trial {r['best_trial']} bucket {r['source_bucket']} buckets {r['buckets_enriched']} exact {ctx.em_exact_counts()}")
    print("planted motif", motif)


if __name__ == "__main__":
    main()
