import sys, time
sys.path.insert(0, '/root/repo')
import paper_1605_06904_b200 as pm
from oracle import pmo
o = pmo.load("port")
ss, motif, pos = o.generate_planted(20, 600, 15, 4, 42)
with pm.Context(0) as ctx:
    for _ in range(5): ctx.set_sequences(ss.bases, ss.offs)
    t0 = time.perf_counter()
    for _ in range(200): ctx.set_sequences(ss.bases, ss.offs)
    print("set_sequences us", (time.perf_counter() - t0) / 200 * 1e6)
