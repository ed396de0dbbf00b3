"""Measured deviation of the CUDA EM path from the reference goldens (theta, expectation, LL trace) -- the numbers
quoted in DESIGN.md section 5."""
import json, os, sys
import numpy as np
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import paper_1605_06904_b200 as pm
from oracle import pmo
golden = json.load(open(os.path.join(REPO, "tests", "golden", "reference_golden.json")))
port = pmo.load("port")
by_inst = {}
for g in golden["refine"]:
    by_inst.setdefault(tuple(g["instance"]), []).append(g)
dth = dex = dll = 0.0
mism = n = 0
with pm.Context(0) as ctx:
    for key, items in by_inst.items():
        ss, _, _ = port.generate_planted(*key)
        ctx.set_sequences(ss.bases, ss.offs)
        got = ctx.refine(items[0]["l"], [g["members"] for g in items])
        for a, g in zip(got, items):
            n += 1
            mism += (a["consensus"], a["positions"], a["score"], a["iterations"]) != (g["consensus"], g["positions"], g["score"], g["iterations"])
            dth = max(dth, float(np.abs(a["theta"].astype(np.float64) - np.asarray(g["theta"])).max()))
            dex = max(dex, abs(a["expectation"] - g["expectation"]))
            k = min(len(a["ll_trace"]), len(g["ll_trace"]))
            dll = max(dll, float(np.abs(np.asarray(a["ll_trace"][:k]) - np.asarray(g["ll_trace"][:k])).max()))
print(f"buckets {n}  discrete mismatches {mism}  max|dtheta| {dth:.3g}  max|dE| {dex:.3g}  max|dLL| {dll:.3g}")
