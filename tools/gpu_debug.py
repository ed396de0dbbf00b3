"""Ad-hoc GPU bring-up script (not a test): stage-by-stage comparison against the oracle."""
import os, sys, time, traceback
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1605_06904_b200 as pm
from oracle import pmo

oracle = pmo.load("reference" if pmo.available("reference") else "port")
print("oracle:", oracle.impl, pm.lib().pm_version())

def stage(name, fn):
    try:
        t0 = time.time(); r = fn(); print(f"[ok] {name} ({time.time()-t0:.3f}s)", r if r is not None else ""); return True
    except Exception as e:
        print(f"[FAIL] {name}: {e}"); traceback.print_exc(); return False

ctx = pm.Context(0)
ss, motif, pos = oracle.generate_planted(20, 600, 15, 4, 42)
ctx.set_sequences(ss.bases, ss.offs)
kept = oracle.trial_plan(15, 7, 7, 1)

def t_pack():
    words, woff = ctx.packed_words()
    strs = ss.strings()
    code = {'A':0,'C':1,'T':2,'G':3}
    for i, s in enumerate(strs):
        for w in range((len(s)+31)//32):
            val = 0
            for p in range(32):
                b = code[s[w*32+p]] if w*32+p < len(s) else 0
                val |= b << (62-2*p)
            assert int(words[woff[i]+w]) == val, (i, w, hex(int(words[woff[i]+w])), hex(val))
    cnt = ctx.symbol_counts()
    full = "".join(strs)
    assert cnt == [full.count('A'), full.count('C'), full.count('T'), full.count('G')], cnt
stage("encode", t_pack)

def t_keys():
    a = ctx.hash_keys(15, kept); b = oracle.hash_keys(ss, 15, kept)
    assert (a == b).all(), np.nonzero(a != b)[0][:10]
stage("hash_keys", t_keys)

def t_trial():
    ka, sa, ma = ctx.hash_trial(15, kept); kb, sb, mb = oracle.hash_trial(ss, 15, kept)
    assert len(ka) == len(kb), (len(ka), len(kb))
    assert (ka == kb).all() and (sa == sb).all() and (ma == mb).all()
    return len(ka)
stage("hash_trial", t_trial)

def t_enr():
    a = ctx.enriched_buckets(15, kept, 4, 80); b = oracle.enriched(ss, 15, kept, 4, 80)
    assert len(a) == len(b), (len(a), len(b))
    assert a == b
    return len(a)
stage("enriched", t_enr)

en = oracle.enriched(ss, 15, kept, 4, 80)
def t_refine():
    got = ctx.refine(15, [e["members"] for e in en])
    bad = 0; maxdt = 0; maxde = 0; maxdll = 0
    for e, g in zip(en, got):
        w = oracle.refine(ss, 15, e["members"], e["key"])
        dt = np.abs(g["theta"].astype(np.float64) - w.theta).max()
        maxdt = max(maxdt, dt); maxde = max(maxde, abs(g["expectation"] - w.expectation))
        if len(g["ll_trace"]) == len(w.ll_trace):
            maxdll = max(maxdll, max(abs(a-b) for a, b in zip(g["ll_trace"], w.ll_trace)))
        if (g["consensus"], g["positions"], g["score"], g["iterations"]) != (w.consensus, w.positions, w.score, w.iterations):
            bad += 1
            if bad < 4: print("  mismatch", g["consensus"], w.consensus, g["score"], w.score, g["iterations"], w.iterations)
    return dict(buckets=len(en), mismatches=bad, max_dtheta=maxdt, max_dexp=maxde, max_dll=maxdll)
stage("refine", t_refine)

def t_refine_dense():
    got = ctx.refine(15, [e["members"] for e in en[:20]], z_epsilon=0.0)
    got2 = ctx.refine(15, [e["members"] for e in en[:20]])
    return max(np.abs(a["theta"] - b["theta"]).max() for a, b in zip(got, got2))
stage("refine eps=0 vs default (max dtheta)", t_refine_dense)

def t_run():
    kw = dict(l=15, d=4, k=7, s=4, m=16, seed=7, early_stop=0)
    t0 = time.time(); got = ctx.run(profile=1, **kw); t1 = time.time()
    want = oracle.run(ss, **kw); t2 = time.time()
    print("  gpu", {k: got[k] for k in ("consensus","score","expectation","source_bucket","best_trial","trials_run","buckets_enriched","within_d","total_distance","gpu_launches","stage_ms","wall_ms")})
    print("  cpu", {k: want[k] for k in ("consensus","score","expectation","source_bucket","best_trial","trials_run","buckets_enriched","wall_ms")})
    assert got["consensus"] == want["consensus"] and got["score"] == want["score"] and got["positions"] == want["positions"]
    assert got["buckets_enriched"] == want["buckets_enriched"] and got["best_trial"] == want["best_trial"]
    return f"gpu {t1-t0:.3f}s cpu {t2-t1:.3f}s"
stage("run m=16", t_run)

def t_run_big():
    kw = dict(l=15, d=4, k=7, s=4, m=172, seed=7, early_stop=0)
    got = ctx.run(profile=1, **kw)
    t0 = time.time(); got = ctx.run(**kw); t1 = time.time()
    print("  gpu", {k: got[k] for k in ("consensus","score","expectation","best_trial","buckets_enriched","gpu_launches","wall_ms","em_lookup_adds")})
    return f"172 trials in {t1-t0:.4f}s -> {172/(t1-t0):.1f} trials/s"
stage("run m=172", t_run_big)

def t_smoke():
    import __graft_entry__ as g
    g.smoke()
stage("smoke", t_smoke)
