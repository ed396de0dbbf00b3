"""world_size-2 gloo test of the multi-GPU path's host side: contiguous trial shards, the
all_gather of the fixed-size result record and pm_merge_results.  On CPU the per-shard results come
from the oracle's per-trial outcomes (the device arm needs a GPU); the merged result must equal
the oracle's single-process run()."""
import os
import socket

import numpy as np
import pytest

from oracle import pmo

CFG = dict(l=8, d=1, k=5, s=3, m=7, seed=3, early_stop=0)
INSTANCE = (12, 120, 8, 1, 5)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, early_stop, queue):
    import torch.distributed as dist
    import paper_1605_06904_b200 as pm
    from paper_1605_06904_b200.sharding import all_gather_merge, shard_range

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        oracle = pmo.load("port")
        ss, _, _ = oracle.generate_planted(*INSTANCE)
        cfg = dict(CFG, early_stop=early_stop)
        begin, end = shard_range(cfg["m"], rank, world)
        part = pm.RunResult()
        part.k, part.s, part.m, part.q, part.t_hat = cfg["k"], cfg["s"], cfg["m"], 0.95, ss.t
        pos = None
        if end >= begin:
            buckets, score, exp_, key = oracle.trial_outcomes(ss, begin, end, **cfg)
            best = None
            for i in range(end - begin + 1):
                part.trials_run = begin + i
                part.buckets_enriched += int(buckets[i])
                cand = (int(score[i]), float(exp_[i]), int(key[i]))
                if score[i] >= 0 and (best is None or pm.candidate_improves(cand, best)):
                    best = cand
                    part.best_trial = begin + i
                if early_stop and best is not None and best[0] == cfg["l"] * ss.t:
                    break
            if best is not None:
                part.found, part.score, part.expectation, part.source_bucket = 1, best[0], best[1], best[2]
                part.consensus = str(part.best_trial).encode()
                pos = np.full(ss.t, part.best_trial, dtype=np.int32)
        merged, mpos = all_gather_merge(part, pos, ss.t, cfg["l"], bool(early_stop))
        queue.put((rank, merged.score, merged.expectation, merged.source_bucket, merged.best_trial, merged.trials_run,
                   merged.buckets_enriched, merged.consensus.decode(), mpos.tolist()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("early_stop", [0, 1])
def test_two_rank_shards_merge_to_the_single_process_result(early_stop):
    import torch.multiprocessing as mp
    oracle = pmo.load("port")
    ss, _, _ = oracle.generate_planted(*INSTANCE)
    want = oracle.run(ss, **dict(CFG, early_stop=early_stop))
    ctx = mp.get_context("spawn")
    queue = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, early_stop, queue)) for r in range(2)]
    for p in procs:
        p.start()
    results = [queue.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for _, score, exp_, key, best_trial, trials_run, buckets, cons, pos in results:
        assert (score, exp_, key, best_trial) == (want["score"], want["expectation"], want["source_bucket"], want["best_trial"])
        assert (trials_run, buckets) == (want["trials_run"], want["buckets_enriched"])
        assert cons == str(want["best_trial"]) and pos == [want["best_trial"]] * ss.t
