import os, sys, time
sys.path.insert(0, os.getcwd())
import paper_1605_06904_b200 as pm
bases, offs, motif, _ = pm.generate_planted(20, 600, 15, 4, 42)
with pm.Context(0) as c:
    c.set_sequences(bases, offs)
    kept = pm.trial_plan(15, 7, 7, 1)
    en = c.enriched_buckets(15, kept, 4, 80)
    for nb in (1, 8, 64):
        lists = [e["members"] for e in en[:nb]]
        c.refine(15, lists, exact=True)
        ts = []
        for _ in range(5):
            t0 = time.perf_counter(); c.refine(15, lists, exact=True); ts.append(time.perf_counter() - t0)
        tp = []
        for _ in range(5):
            t0 = time.perf_counter(); c.refine(15, lists); tp.append(time.perf_counter() - t0)
        print(f"C1 buckets={nb}: pm_refine_exact {min(ts)*1e3:.3f} ms wall, pm_refine (pair) {min(tp)*1e3:.3f} ms wall")
