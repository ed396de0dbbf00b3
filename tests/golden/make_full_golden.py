"""Generates tests/golden/reference_full_<cfg>.json: challenge-scale known answers for every BASELINE
configuration, from the UNMODIFIED reference (oracle/_ref/libpm_ref.so, built by oracle/Makefile).

    python tests/golden/make_full_golden.py [c1 c2 c3 c3b c4] [--procs N]

Build container only (hours of CPU for all five: a (20,7) trial costs ~5 s of one core and there are
3,421 of them).  Per configuration the fixture holds
  * the instance pin (SHA-256 of generate_planted(t,n,l,d,42)), the resolved k/s/m;
  * `outcomes`: for EVERY trial 1..m the reference's run_trial view (driver.hpp:163-177):
    enriched-bucket count, best score, best expectation, best bucket key;
  * `run`: the RunResult of run(m, seed=7, early_stop=false).  Obtained by the reference's own ascending
    scan (driver.hpp:195-203) over the outcomes plus one reference refine() of the winning bucket; for
    c1 and c3b the same record also comes from a direct reference run() and must agree (checked here);
  * `hash`: SHA entries of trial 1's keys / grouping and its full enriched list;
  * `refine`: >= 50 refined buckets (every n-th enriched bucket of trials 1 and m).
"""
import hashlib
import json
import multiprocessing as mp
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle import pmo  # noqa: E402

CONFIGS = {  # SURVEY.md section 8(d); k=7, s=4 overrides, instance seed 42, run seed 7
    "c1": dict(t=20, n=600, l=15, d=4, m=172),
    "c2": dict(t=20, n=1000, l=16, d=5, m=1293),
    "c3": dict(t=20, n=1000, l=18, d=6, m=2218),
    "c3b": dict(t=20, n=1000, l=19, d=6, m=711),
    "c4": dict(t=20, n=1000, l=20, d=7, m=3421),
}
DIRECT_RUN = ("c1", "c3b")
K, S, INST_SEED, RUN_SEED = 7, 4, 42, 7


def sha(b):
    return hashlib.sha256(b).hexdigest()


def _chunk(args):
    name, lo, hi = args
    c = CONFIGS[name]
    ref = pmo.load("reference")
    ss, _, _ = ref.generate_planted(c["t"], c["n"], c["l"], c["d"], INST_SEED)
    b, s, e, k = ref.trial_outcomes(ss, lo, hi, l=c["l"], d=c["d"], k=K, s=S, m=c["m"], seed=RUN_SEED, early_stop=0)
    return lo, b.tolist(), s.tolist(), [float(v) for v in e], [int(v) for v in k]


def improves(a, b):
    """detail::candidate_improves (driver.hpp:127-135) on (score, expectation, key)."""
    if a[0] != b[0]:
        return a[0] > b[0]
    if a[1] != b[1]:
        return a[1] > b[1]
    return a[2] < b[2]


def make(name, procs):
    c = CONFIGS[name]
    ref = pmo.load("reference")
    assert ref.impl == "reference"
    l, d, m = c["l"], c["d"], c["m"]
    ss, motif, pos = ref.generate_planted(c["t"], c["n"], l, d, INST_SEED)
    params = ref.resolve_params(ss, l=l, d=d, k=K, s=S, seed=RUN_SEED)
    assert params["m"] == m, (params, m)
    g = dict(config=name, instance=[c["t"], c["n"], l, d, INST_SEED], sha256=sha(ss.bases), motif=motif,
             planted_positions=pos, k=K, s=S, m=m, seed=RUN_SEED)

    t0 = time.time()
    step = 4
    jobs = [(name, lo, min(lo + step - 1, m)) for lo in range(1, m + 1, step)]
    out = dict(buckets=[0] * m, score=[0] * m, expectation=[0.0] * m, key=[0] * m)
    with mp.Pool(procs) as pool:
        for n_done, (lo, b, s, e, k) in enumerate(pool.imap_unordered(_chunk, jobs)):
            out["buckets"][lo - 1:lo - 1 + len(b)] = b
            out["score"][lo - 1:lo - 1 + len(b)] = s
            out["expectation"][lo - 1:lo - 1 + len(b)] = e
            out["key"][lo - 1:lo - 1 + len(b)] = k
            if n_done % 50 == 0:
                print(f"[{name}] {n_done}/{len(jobs)} chunks, {time.time() - t0:.0f} s", flush=True)
    g["outcomes"] = out

    best = None
    for tr in range(1, m + 1):
        if out["score"][tr - 1] < 0:
            continue
        cand = (out["score"][tr - 1], out["expectation"][tr - 1], out["key"][tr - 1], tr)
        if best is None or improves(cand, best):
            best = cand
    kept = ref.trial_plan(l, K, RUN_SEED, best[3])
    en = ref.enriched(ss, l, kept, S, c["t"] * S)
    win = [e for e in en if e["key"] == best[2]][0]
    cand = ref.refine(ss, l, win["members"], win["key"])
    assert cand.score == best[0] and cand.expectation == best[1]
    g["run"] = dict(consensus=cand.consensus, score=cand.score, iterations=cand.iterations, expectation=cand.expectation,
                    source_bucket=best[2], best_trial=best[3], trials_run=m, buckets_enriched=int(sum(out["buckets"])),
                    k=K, s=S, m=m, positions=cand.positions)
    g["run_source"] = "ascending scan of outcomes + refine of the winner"
    if name in DIRECT_RUN:
        r = ref.run(ss, l=l, d=d, k=K, s=S, m=m, seed=RUN_SEED, early_stop=0, workers=procs)
        for f in ("consensus", "score", "iterations", "expectation", "source_bucket", "best_trial", "trials_run",
                  "buckets_enriched", "positions"):
            assert r[f] == g["run"][f], (f, r[f], g["run"][f])
        g["run_source"] = "direct reference run(), identical to the scan of outcomes"

    g["hash"] = []
    g["refine"] = []
    for tr in (1, m):
        kept = ref.trial_plan(l, K, RUN_SEED, tr)
        hk = ref.hash_keys(ss, l, kept)
        bk, bs, bm = ref.hash_trial(ss, l, kept)
        en = ref.enriched(ss, l, kept, S, c["t"] * S)
        g["hash"].append(dict(trial=tr, kept=kept, keys_sha256=sha(hk.astype("<u8").tobytes()), n_buckets=int(len(bk)),
                              bucket_keys_sha256=sha(bk.astype("<u8").tobytes()),
                              bucket_sizes_sha256=sha(bs.astype("<i4").tobytes()),
                              members_sha256=sha(bm.astype("<i4").tobytes()),
                              enriched=en if tr == 1 else None, n_enriched=len(en)))
        stride = max(1, len(en) // 28)
        for e in en[::stride]:
            cd = ref.refine(ss, l, e["members"], e["key"])
            g["refine"].append(dict(trial=tr, members=e["members"], key=e["key"], consensus=cd.consensus,
                                    positions=cd.positions, score=cd.score, expectation=cd.expectation,
                                    iterations=cd.iterations, theta=cd.theta.tolist(), ll_trace=cd.ll_trace))
    path = os.path.join(HERE, f"reference_full_{name}.json")
    with open(path, "w") as f:
        json.dump(g, f, separators=(",", ":"))
    print(f"[{name}] wrote {path} ({os.path.getsize(path)} B) in {time.time() - t0:.0f} s; run = {g['run']}", flush=True)


if __name__ == "__main__":
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    procs = 6
    if "--procs" in sys.argv:
        procs = int(sys.argv[sys.argv.index("--procs") + 1])
        args = [a for a in args if a != str(procs)]
    for name in (args or list(CONFIGS)):
        make(name, procs)
