"""C5 (t=10,000 x n=1000, (15,4)) bring-up: hashing/enrichment bit-exact vs the oracle, a few buckets'
EM vs the oracle, then a timed 2-trial run."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1605_06904_b200 as pm
from oracle import pmo

port = pmo.load("port")
t0 = time.time(); bases, offs, motif, pos = pm.generate_planted(10000, 1000, 15, 4, 42); print("generate", time.time() - t0)
ss = pmo.SeqSet(bases, offs)
ctx = pm.Context(0)
t0 = time.time(); ctx.set_sequences(bases, offs); print("set_sequences (upload+encode+class tables)", time.time() - t0)
l, k, s = 15, 10, 19
kept = pm.trial_plan(l, k, 7, 1)
t0 = time.time(); gk = ctx.hash_keys(l, kept); t1 = time.time(); ok = port.hash_keys(ss, l, kept); t2 = time.time()
print("hash_keys gpu %.3fs cpu %.3fs equal=%s" % (t1 - t0, t2 - t1, bool((gk == ok).all())))
t0 = time.time(); ge = ctx.enriched_buckets(l, kept, s, 10000 * s); t1 = time.time(); oe = port.enriched(ss, l, kept, s, 10000 * s); t2 = time.time()
print("enriched gpu %.3fs cpu %.3fs n=%d equal=%s" % (t1 - t0, t2 - t1, len(ge), ge == oe))
pick = [oe[0], oe[len(oe) // 2]]
t0 = time.time(); got = ctx.refine(l, [e["members"] for e in pick]); t1 = time.time()
print("refine 2 buckets gpu %.3fs" % (t1 - t0))
for e, a in zip(pick, got):
    t0 = time.time(); w = port.refine(ss, l, e["members"], e["key"]); dt = time.time() - t0
    same = (a["consensus"], a["score"], a["iterations"], a["positions"]) == (w.consensus, w.score, w.iterations, w.positions)
    npos = sum(1 for x, y in zip(a["positions"], w.positions) if x != y)
    print("  bucket key=%d size=%d cpu %.1fs discrete_equal=%s pos_mismatch=%d dtheta=%.2e dE=%.2e score %d/%d" % (
        e["key"], e["size"], dt, same, npos, np.abs(a["theta"] - w.theta).max(), abs(a["expectation"] - w.expectation), a["score"], w.score))
for m in (1, 2):
    t0 = time.time(); r = ctx.run(l=l, d=4, k=k, s=s, m=m, seed=7, early_stop=0, profile=1); dt = time.time() - t0
    print("run m=%d: %.2fs -> %.3f trials/s  buckets=%d score=%d consensus=%s motif=%s stage_ms=%s" % (
        m, dt, m / dt, r["buckets_enriched"], r["score"], r["consensus"], motif, [round(x, 1) for x in r["stage_ms"]]))
