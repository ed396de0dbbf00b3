"""Generates tests/golden/*.json by running the UNMODIFIED reference (oracle/_ref/libpm_ref.so, built
from /root/reference by oracle/Makefile).  Run in the build container only:

    python tests/golden/make_golden.py

The fixtures are what travels to the GPU box (where /root/reference does not exist); tests compare
the C oracle and the CUDA path against them.  Sequences are not stored: instances are regenerated
by generate_planted and pinned by the SHA-256 recorded here.
"""
import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle import pmo  # noqa: E402

EXAMPLE = [
    "CGGGGCTATGGAACTGGGTCGTCACATTCCCCTTTCGATA", "TTTGAGGGTGCCCAATAAATGCCACTCCAAAGCGGACAAA",
    "GGATGCAACTGATGCCGTTTGACGACCTAAATCAACGGCC", "AAGGATGCAACTCCAGGAGCGCCTTTGCTGGTTCTACCTG",
    "AATTTTCTAAAAAGATTATAATGTCGGTCCATGCAACTTC", "CTGCTGTACAACTGAGATCATGCTGCATGCAACTTTCAAC",
    "TACATGATCTTTTGATGCAACGTGGATGAGGGAATGATGC",
]


def sha(b):
    return hashlib.sha256(b).hexdigest()


def cand_dict(c):
    return dict(consensus=c.consensus, positions=c.positions, score=c.score, expectation=c.expectation,
                iterations=c.iterations, theta=c.theta.tolist(), ll_trace=c.ll_trace)


def main():
    ref = pmo.load("reference")
    assert ref.impl == "reference"
    g = {}

    # ---- PRNG stream (rng.hpp)
    g["derive_seed"] = [[m, i, ref.derive_seed(m, i)] for m in (0, 7, 42, 2**63 + 5) for i in (0, 1, 2, 1000)]
    g["mt_outputs"] = [[s, ref.mt_outputs(s, 5).tolist()] for s in (0, 1, ref.derive_seed(7, 1))]
    g["uniform_below"] = [[s, b, ref.uniform_below(s, b, 8).tolist()] for s in (3, 99) for b in (1, 2, 15, 1000, 2**63 + 1)]
    g["plans"] = [dict(l=l, k=k, master=ms, trial=tr, kept=ref.trial_plan(l, k, ms, tr))
                  for (l, k) in ((15, 7), (16, 7), (18, 7), (20, 7), (15, 10), (8, 5), (9, 9), (31, 17), (4, 1))
                  for ms in (0, 7) for tr in (1, 2, 3, 172)]

    # consecutive plans from one generator (sample_plan consumes the caller's Rng, projection.hpp:210-226)
    g["plans_consecutive"] = [dict(l=l, k=k, seed=sd, plans=ref.sample_plans(l, k, sd, 4))
                              for (l, k) in ((15, 7), (20, 7), (9, 9), (31, 17)) for sd in (0, 12345)]

    # ---- formulas (projection.hpp:97-206)
    g["p_hat"] = [[l, d, k, ref.p_hat(l, d, k)] for (l, d) in ((15, 4), (16, 5), (18, 6), (19, 6), (20, 7), (8, 1))
                  for k in (0, 1, 5, 7, l - d, l - d + 1 if l - d + 1 <= l else l)]
    g["binomial_lt"] = [[t, p, s, ref.binomial_lt(t, p, s)] for t in (1, 7, 20) for p in (0.0, 0.01, 0.2, 0.5, 1.0)
                        for s in (0, 1, 3, 4, 21)]
    g["num_trials"] = [[l, d, ref.num_trials(0.95, 20, ref.p_hat(l, d, 7), 4)]
                       for (l, d) in ((14, 4), (15, 4), (16, 5), (18, 6), (19, 6), (20, 7))]
    g["bucket_threshold"] = [[w, k, f, ref.bucket_threshold_for_windows(w, k, f)]
                             for (w, k, f) in ((11720, 10, 3), (11720, 7, 3), (9860000, 10, 3), (9860000, 7, 3), (231, 5, 3), (10**6, 4, 1))]

    # ---- planted instances (planted.hpp:38-101)
    insts = {}
    g["planted"] = []
    for (t, n, l, d, seed) in ((20, 600, 15, 4, 42), (20, 1000, 16, 5, 42), (12, 120, 8, 1, 5), (8, 60, 9, 2, 1234),
                               (5, 50, 10, 0, 77), (6, 30, 5, 0, 99), (4, 30, 8, 2, 3), (6, 60, 31, 1, 11)):
        ss, motif, pos = ref.generate_planted(t, n, l, d, seed)
        insts[(t, n, l, d, seed)] = ss
        g["planted"].append(dict(t=t, n=n, l=l, d=d, seed=seed, motif=motif, positions=pos, sha256=sha(ss.bases),
                                 head=ss.bases[:30].decode()))

    # ---- worked example (tests/support.hpp:20-54, test_projection.cpp:171-197, test_refine.cpp:154-163)
    ex = pmo.SeqSet.from_strings(EXAMPLE)
    kept = [1, 2, 3, 6, 7]
    en = ref.enriched(ex, 8, kept, 4, 28)
    keys, sizes, members = ref.hash_trial(ex, 8, kept)
    g["worked"] = dict(
        kept=kept, n_buckets=int(len(keys)), keys=[int(v) for v in keys], sizes=sizes.tolist(), members=members.tolist(),
        enriched_s4=en, enriched_s4_cap5=ref.enriched(ex, 8, kept, 4, 5), enriched_s1=ref.enriched(ex, 8, kept, 1, 7 * 33),
        theta0=ref.init_model(ex, 8, en[0]["members"]).tolist(),
        refine=cand_dict(ref.refine(ex, 8, en[0]["members"], en[0]["key"])),
        run=ref.run(ex, l=8, d=1, s=4, forced_kept=kept),
        score=ref.score(ex, 8, [8, 19, 3, 5, 31, 27, 15]),
        total_distance=ref.total_distance(ex, "ATGCAACT"),
    )
    for r in (g["worked"]["run"],):
        r.pop("wall_ms")

    # ---- challenge-scale hashing / enrichment (C1, first three trials; C2 first trial)
    g["hash"] = []
    for key_, l, k, s, trials in (((20, 600, 15, 4, 42), 15, 7, 4, (1, 2, 3)), ((20, 1000, 16, 5, 42), 16, 7, 4, (1,)),
                                  ((20, 600, 15, 4, 42), 15, 10, 3, (1,))):
        ss = insts[key_]
        for tr in trials:
            kept = ref.trial_plan(l, k, 7, tr)
            hk = ref.hash_keys(ss, l, kept)
            bk, bs, bm = ref.hash_trial(ss, l, kept)
            en = ref.enriched(ss, l, kept, s, ss.t * s)
            g["hash"].append(dict(instance=list(key_), l=l, k=k, s=s, trial=tr, kept=kept,
                                  keys_sha256=sha(hk.astype("<u8").tobytes()), n_buckets=int(len(bk)),
                                  bucket_keys_sha256=sha(bk.astype("<u8").tobytes()),
                                  bucket_sizes_sha256=sha(bs.astype("<i4").tobytes()),
                                  members_sha256=sha(bm.astype("<i4").tobytes()), enriched=en))

    # ---- refine goldens: every 6th enriched bucket of C1 trial 1 and of C2 trial 1
    g["refine"] = []
    for h in g["hash"]:
        if h["k"] != 7 or h["trial"] != 1:
            continue
        ss = insts[tuple(h["instance"])]
        for e in h["enriched"][::6]:
            c = ref.refine(ss, h["l"], e["members"], e["key"])
            g["refine"].append(dict(instance=h["instance"], l=h["l"], members=e["members"], key=e["key"], **cand_dict(c)))

    # ---- em_step golden on a generic (non-bucket) model
    ss = insts[(12, 120, 8, 1, 5)]
    th0 = ref.init_model(ss, 8, [3, 200, 411], 0.5)
    th1, ll = ref.em_step(ss, 8, th0)
    g["em_step"] = dict(instance=[12, 120, 8, 1, 5], l=8, members=[3, 200, 411], pseudocount=0.5, theta0=th0.tolist(),
                        theta1=th1.tolist(), ll=ll)

    # ---- whole runs (driver.hpp:145-220)
    g["run"] = []
    runs = [
        ((20, 600, 15, 4, 42), dict(l=15, d=4, k=7, s=4, m=16, seed=7, early_stop=0)),
        ((20, 1000, 16, 5, 42), dict(l=16, d=5, k=7, s=4, m=2, seed=7, early_stop=0)),
        ((12, 120, 8, 1, 5), dict(l=8, d=1, k=5, s=3, m=6, seed=3, early_stop=0)),
        ((8, 60, 9, 2, 1234), dict(l=9, d=2, seed=42)),                       # test_driver.cpp:124-151 (defaults)
        ((5, 50, 10, 0, 77), dict(l=10, d=0, seed=5, m=10)),                  # early stop, test_driver.cpp:104-122
        ((5, 50, 10, 0, 77), dict(l=10, d=0, seed=5, m=10, early_stop=0)),
        ((6, 60, 31, 1, 11), dict(l=31, d=1, k=17, s=2, m=4, seed=1, early_stop=0)),  # widest l, 64-bit keys
    ]
    for key_, kw in runs:
        r = ref.run(insts[key_], **kw)
        r.pop("wall_ms")
        g["run"].append(dict(instance=list(key_), cfg=kw, result=r))
    b, s, e, k = ref.trial_outcomes(insts[(20, 600, 15, 4, 42)], 1, 16, l=15, d=4, k=7, s=4, m=16, seed=7, early_stop=0)
    g["trial_outcomes_c1"] = dict(buckets=b.tolist(), score=s.tolist(), expectation=e.tolist(), key=[int(v) for v in k])

    out = os.path.join(HERE, "reference_golden.json")
    with open(out, "w") as f:
        json.dump(g, f, separators=(",", ":"))
    print("wrote", out, os.path.getsize(out), "bytes")


if __name__ == "__main__":
    main()
