import os, sys, time
sys.path.insert(0, '/root/repo')
import paper_1605_06904_b200 as pm
for name,(t,n,l,d,m) in {"c2":(20,1000,16,5,400),"c1":(20,600,15,4,172)}.items():
    bases, offs, motif, _ = pm.generate_planted(t, n, l, d, 42)
    with pm.Context(0) as ctx:
        ctx.set_sequences(bases, offs)
        kw = dict(l=l, d=d, k=7, s=4, m=m, seed=7, early_stop=0, profile=1)
        r = ctx.run(**kw)
        ts=[]
        for _ in range(3):
            t0=time.time(); r=ctx.run(**kw); ts.append(time.time()-t0)
        print(name, "wall %.2f ms em %.2f ms fp64 buckets %d exact %d" % (min(ts)*1e3, r['stage_ms'][3], r['em_fp64_buckets'], r['em_exact_buckets']), r['stage_ms'])
