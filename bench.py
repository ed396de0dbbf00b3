#!/usr/bin/env python
"""bench.py — projection trials/sec of the PROJECTION hot path on B200 (BASELINE.json metric).

    python bench.py --gpus 1 --steps 20 --warmup 5             # our arm (CUDA path through the C ABI)
    python bench.py --impl reference --steps 3 --warmup 1      # the reference's CPU path on the host cores
    python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N ...   # N ranks, trial shards

A step = one full pass of the hot path (hash -> bucket -> EM-refine -> score -> reduce) over one
batch of projection trials on synthetic planted-(l,d) data: by default config C1 of BASELINE.json
(the (15,4) instance the metric names): t=20 x n=600, k=7, s=4, m=172 trials (the reference's own
trial count for q=0.95), instance seed 42, run seed 7, early_stop off.  With N ranks every rank
runs its own contiguous shard of N*m trials (weak scaling; --scaling strong shards the config's own m) and
the per-rank bests are merged with one all_gather (NCCL) inside the timed step.
Prints ONE JSON line (see DESIGN.md §7 for every key).
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import threading
import time

REPO = os.path.dirname(os.path.abspath(__file__))
if REPO not in sys.path:
    sys.path.insert(0, REPO)

METRIC = "projection trials/sec"
UNIT = "trials/s"

# BASELINE.json configs: name -> (t, n, l, d, k, s, m from the reference formula)
CONFIGS = {
    "c1": dict(t=20, n=600, l=15, d=4, k=7, s=4, m=172, label="C1 planted (15,4) t=20 n=600 k=7 s=4"),
    "c2": dict(t=20, n=1000, l=16, d=5, k=7, s=4, m=1293, label="C2 planted (16,5) t=20 n=1000 k=7 s=4"),
    "c3": dict(t=20, n=1000, l=18, d=6, k=7, s=4, m=2218, label="C3 planted (18,6) t=20 n=1000 k=7 s=4"),
    "c3b": dict(t=20, n=1000, l=19, d=6, k=7, s=4, m=711, label="C3b planted (19,6) t=20 n=1000 k=7 s=4"),
    "c4": dict(t=20, n=1000, l=20, d=7, k=7, s=4, m=3421, label="C4 planted (20,7) t=20 n=1000 k=7 s=4"),
    # large-scale sweep; k, s are what the reference derives for this size (k=l-d-1, s=ceil(2x/4^k)); m explicit
    "c5": dict(t=10000, n=1000, l=15, d=4, k=10, s=19, m=2, label="C5 planted (15,4) t=10000 n=1000 k=10 s=19",
               extrapolate_cpu=True),
    # the same set with the t=20 configurations' k, s: every one of the 16,384 buckets is enriched (~600 members each)
    "c5b": dict(t=10000, n=1000, l=15, d=4, k=7, s=4, m=1, label="C5b planted (15,4) t=10000 n=1000 k=7 s=4",
                extrapolate_cpu=True),
}
INSTANCE_SEED = 42
RUN_SEED = 7


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="c1", choices=sorted(CONFIGS))
    ap.add_argument("--trials", type=int, default=0, help="trials per step per GPU (default: the config's formula m)")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="weak: N*m trials per step, m per GPU; strong: the config's m trials sharded over the N GPUs")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="skip time-to-motif and the other-config sweep")
    return ap.parse_args()


# ------------------------------------------------------------------------------------------------
# clocks: sampled with nvidia-smi DURING the timed region (B200_PROFILING.md recipe)
# ------------------------------------------------------------------------------------------------
class ClockSampler:
    """nvidia-smi in loop mode, started BEFORE the warm-up (its first row takes ~100 ms) so that rows exist by the time
    the timed region begins; only rows that arrived between mark_begin() and stop() are reported.  A C1 step is about a
    millisecond, 20 of them with their L2 flushes ~50 ms: at one row per 10 ms that is a handful of samples."""
    QUERY = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.rows = []
        self.proc = None
        self.gpu_index = gpu_index
        self.t_begin = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.QUERY}", "--format=csv,noheader,nounits", "-lms", "10",
                 "-i", str(self.gpu_index)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append((time.perf_counter(), [c.strip() for c in line.split(",")]))

    def mark_begin(self):
        self.t_begin = time.perf_counter()

    def stop(self):
        t_end = time.perf_counter()
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        # a row describes the interval before it arrived: accept rows up to one period after the region's end
        inside = [r for ts, r in self.rows if self.t_begin is None or (self.t_begin <= ts <= t_end + 0.02)]
        for r in inside:
            if len(r) < 9:
                continue
            try:
                sm.append(float(r[1]))
                smax.append(float(r[2]))
            except ValueError:
                continue
            for name, val in zip(names, r[5:9]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm), "rows_total": len(self.rows)}


def measured_peaks():
    path = os.path.join(REPO, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            p = json.load(f)
        return p.get("hbm_gbs", 6650.0), p.get("sm_max_mhz", 1965.0), "measured", p.get("bf16_tflops", 1590.0)
    return 6650.0, 1965.0, "fallback", 1590.0


def workload_config(cfg, trials_per_step, world, scaling):
    """The `config` object of the JSON line: identical for both arms (what was run, not how)."""
    return {"workload": cfg["label"], "trials_per_step": trials_per_step, "instance_seed": INSTANCE_SEED,
            "run_seed": RUN_SEED, "early_stop": False, "n_gpus": world, "scaling_mode": scaling}


def recorded_traffic(kernel, config_name):
    """DRAM bytes per launch of `kernel` from the ncu --set full capture summarised in profiles/traffic.json
    (written by tools/ncu_traffic.py together with the commit it was taken at); None when there is no capture."""
    path = os.path.join(REPO, "profiles", "traffic.json")
    if not os.path.exists(path):
        return None, None
    with open(path) as f:
        rec = json.load(f)
    for r in rec.get("captures", []):
        if r.get("kernel") == kernel and r.get("config") == config_name:
            return r.get("dram_bytes_per_launch"), f"profiles/traffic.json: {r.get('report')} at commit {r.get('commit')}"
    return None, None


# ------------------------------------------------------------------------------------------------
# the reference arm / cpu_baseline: the reference's own CPU implementation on the host cores
# ------------------------------------------------------------------------------------------------
def load_cpu_oracle():
    from oracle import pmo
    kind = "reference" if pmo.available("reference") else "port"
    return pmo.load(kind), kind


def cpu_trials_per_second(oracle, kind, ss, cfg, trials, workers):
    """Times run() of the reference on `trials` trials of the workload (bounded sample)."""
    t0 = time.perf_counter()
    oracle.run(ss, l=cfg["l"], d=cfg["d"], k=cfg["k"], s=cfg["s"], m=trials, seed=RUN_SEED, early_stop=0,
               workers=workers)
    dt = time.perf_counter() - t0
    return trials / dt, dt


def cpu_extrapolated_trials_per_second(oracle, ss, cfg, workers, n_buckets_sample=16):
    """C5: a full CPU trial is hours.  Time hash_trial+enriched_buckets of one trial in full and
    refine() on a sample of its buckets (spread over `workers` threads), then extrapolate:
    trial time = t_hash + n_buckets * mean(t_refine) / workers.  Labelled as extrapolated."""
    from concurrent.futures import ThreadPoolExecutor
    kept = oracle.trial_plan(cfg["l"], cfg["k"], RUN_SEED, 1)
    t0 = time.perf_counter()
    en = oracle.enriched(ss, cfg["l"], kept, cfg["s"], ss.t * cfg["s"])
    t_hash = time.perf_counter() - t0
    step = max(1, len(en) // n_buckets_sample)
    pick = en[::step][:n_buckets_sample]

    def one(e):
        a = time.perf_counter()
        oracle.refine(ss, cfg["l"], e["members"], e["key"], want_theta=False)
        return time.perf_counter() - a
    t0 = time.perf_counter()
    with ThreadPoolExecutor(max_workers=workers) as ex:
        per = list(ex.map(one, pick))
    wall = time.perf_counter() - t0
    t_trial = t_hash + len(en) * (sum(per) / len(per)) / workers
    return 1.0 / t_trial, dict(t_hash_s=t_hash, buckets=len(en), refine_s_mean=sum(per) / len(per), sampled=len(pick),
                               sample_wall_s=wall + t_hash)


def run_reference_arm(args, cfg, rank, world):
    if rank != 0:
        return  # rank 0 alone runs the CPU arm
    oracle, kind = load_cpu_oracle()
    ss, _, _ = oracle.generate_planted(cfg["t"], cfg["n"], cfg["l"], cfg["d"], INSTANCE_SEED)
    cores = os.cpu_count() or 1
    workers = cores if kind == "reference" else 1  # the C port is a scalar single-thread restatement
    if cfg.get("extrapolate_cpu"):
        vals, info = [], None
        for _ in range(max(1, min(args.steps, 2))):
            v, info = cpu_extrapolated_trials_per_second(oracle, ss, cfg, cores)
            vals.append(v)
        value = sum(vals) / len(vals)
        line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": len(vals),
                "warmup": 0, "ms_per_step": 1e3 / value, "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None,
                "dtype": "f64", "data": "synthetic",
                "config": dict(workload_config(cfg, (args.trials or cfg["m"]) * (world if args.scaling == "weak" else 1), world, args.scaling),
                               note="EXTRAPOLATED: hashing in full + refine() on sampled buckets, see cpu_baseline.sample"),
                "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": kind,
                                 "sample": f"extrapolated from {info}"},
                "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}, "gpu_launches": 0}
        print(json.dumps(line), flush=True)
        return
    # One step = the step of our arm: the config's own m trials (x N for the weak-scaling runs).  That is ~2.5 s of the
    # host's 16 cores on C1; the n = 1000 configurations need minutes per step, so they run a bounded sample of the
    # same trials instead (trial cost is i.i.d.) and say so.
    want = (args.trials or cfg["m"]) * (world if args.scaling == "weak" else 1)
    calib, dt = cpu_trials_per_second(oracle, kind, ss, cfg, max(workers, 2), workers)
    budget_s = max(2.0, 150.0 / max(1, args.steps + args.warmup))  # the whole arm ends within a few minutes
    sample = want if want / calib <= budget_s else max(workers, int(calib * budget_s) // workers * workers)
    for _ in range(args.warmup if sample < want else min(args.warmup, 1)):
        cpu_trials_per_second(oracle, kind, ss, cfg, sample, workers)
    times = []
    for _ in range(args.steps):
        _, dt = cpu_trials_per_second(oracle, kind, ss, cfg, sample, workers)
        times.append(dt)
    total = sum(times)
    value = sample * args.steps / total
    config = workload_config(cfg, want, world, args.scaling)
    if sample != want:
        config["reference_sample_trials_per_step"] = sample
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps * (want / sample), "higher_is_better": True,
        "scaling": args.scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": config,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": workers, "kind": kind,
                         "sample": f"{sample} trials/step x {args.steps} steps of projmotif::run "
                                   f"(-O3, workers={workers}) on {cores} host cores"
                                   + ("" if sample == want else f"; bounded sample of the step's {want} trials")},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------------------------
# our arm
# ------------------------------------------------------------------------------------------------
def run_b200_arm(args, cfg, rank, world, local_rank):
    import numpy as np
    import torch

    import paper_1605_06904_b200 as pm
    from paper_1605_06904_b200.sharding import all_gather_merge, shard_range

    if not torch.cuda.is_available():
        raise SystemExit("bench.py --impl b200 needs a B200: the CUDA path has no CPU fallback")
    torch.cuda.set_device(local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist_mod
        dist = dist_mod
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))

    m_per_gpu = args.trials or cfg["m"]
    m_total = m_per_gpu * world if args.scaling == "weak" else m_per_gpu
    begin, end = shard_range(m_total, rank, world)
    stream = torch.cuda.current_stream()
    ctx = pm.Context(local_rank, stream.cuda_stream)

    # synthetic planted instance: the library's host generator (planted.hpp draw order, pinned to the
    # reference by tests/test_host_abi.py), outside every timed region.  This arm never touches oracle/.
    class Inst:
        pass
    ss = Inst()
    ss.bases, ss.offs, motif, _ = pm.generate_planted(cfg["t"], cfg["n"], cfg["l"], cfg["d"], INSTANCE_SEED)
    ss.t = cfg["t"]
    ss.total_lmers = lambda l_: cfg["t"] * (cfg["n"] - l_ + 1)
    t, l = ss.t, cfg["l"]
    kw = dict(l=l, d=cfg["d"], k=cfg["k"], s=cfg["s"], m=m_total, seed=RUN_SEED, early_stop=0,
              trial_begin=begin, trial_end=end, profile=1)

    # pinned host copies of the inputs for the e2e leg
    pinned = torch.empty(len(ss.bases), dtype=torch.uint8).pin_memory()
    pinned.numpy()[:] = np.frombuffer(ss.bases, dtype=np.uint8)
    bases_ptr = C.cast(pinned.data_ptr(), C.c_char_p)
    offs = np.ascontiguousarray(ss.offs, dtype=np.int64)

    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")  # > 126 MB L2

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    def one_step(e2e):
        """One pass over this rank's trial shard + the cross-rank reduction.  Returns the merged result."""
        cfg_c = pm.default_config(**kw)
        out = pm.RunResult()
        pos = np.zeros(t, dtype=np.int32)
        if e2e:
            rc = pm.lib().pm_run_host(ctx._h, C.byref(cfg_c), bases_ptr, offs.ctypes.data_as(C.POINTER(C.c_int64)), t,
                                      C.byref(out), pos.ctypes.data_as(C.POINTER(C.c_int32)))
        else:
            rc = pm.lib().pm_run(ctx._h, C.byref(cfg_c), C.byref(out), pos.ctypes.data_as(C.POINTER(C.c_int32)),
                                 None, None, None, None)
        if rc not in (0, 7):  # a shard may legitimately find no enriched bucket
            raise pm.PmError(rc, pm.lib().pm_last_error().decode())
        if dist is not None:
            merged, mpos = all_gather_merge(out, pos, t, l, False, device=torch.device("cuda", local_rank))
            return out, merged
        return out, out

    def timed_loop(steps, e2e):
        per_step_ms, launches, stage, lookups, h2d, d2h, work = [], 0, [0.0] * 8, 0, 0, 0, 0
        tensor_flops = exact_buckets = fp64_buckets = 0
        result = None
        for _ in range(steps):
            flush.fill_(1)  # evict L2 between timed iterations (untimed)
            barrier()
            ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ev0.record(stream)
            mine, result = one_step(e2e)
            ev1.record(stream)
            barrier()
            ms = torch.tensor([ev0.elapsed_time(ev1)], device="cuda", dtype=torch.float64)
            if dist is not None:
                dist.all_reduce(ms, op=dist.ReduceOp.MAX)  # device-timed, max over ranks
            per_step_ms.append(float(ms.item()))
            launches += mine.gpu_launches
            lookups += mine.em_lookup_adds
            work += mine.em_work
            tensor_flops += mine.em_tensor_flops
            exact_buckets += mine.em_exact_buckets
            fp64_buckets += mine.em_fp64_buckets
            h2d += mine.h2d_bytes
            d2h += mine.d2h_bytes
            for i in range(8):
                stage[i] += mine.stage_ms[i]
        return per_step_ms, launches, stage, lookups, h2d, d2h, result, work, (tensor_flops, exact_buckets, fp64_buckets)

    ctx.set_sequences(ss.bases, ss.offs)
    sampler = ClockSampler(local_rank)
    if rank == 0:
        sampler.start()                                 # running before the warm-up: rows exist when the timed region begins
    timed_loop(args.warmup, False)                      # warm-up (untimed)
    sampler.mark_begin()
    ms_dev, launches, stage, lookups, _, _, result, work, (tensor_flops, exact_buckets, fp64_buckets) = timed_loop(args.steps, False)
    timed_loop(max(1, min(args.warmup, 2)), True)
    ms_e2e, _, stage_e2e, _, h2d, d2h, result_e2e, _, _ = timed_loop(args.steps, True)
    clocks = sampler.stop() if rank == 0 else None  # sampled across both timed loops (HBM-resident and end-to-end)

    # time to the planted motif on N GPUs: round-robin trial shards (every rank takes part)
    ttm_multi = None
    if not args.no_extras and cfg["t"] <= 100 and world > 1:
        ttm_multi = time_to_motif_sharded(pm, ctx, cfg, dist, rank, world, torch.device("cuda", local_rank), all_gather_merge)

    if rank != 0:
        if dist is not None:
            dist.destroy_process_group()
        return

    mean_ms = sum(ms_dev) / len(ms_dev)
    value = m_total / (mean_ms * 1e-3)
    mean_e2e = sum(ms_e2e) / len(ms_e2e)
    hbm_peak, sm_max_mhz, peak_kind, bf16_peak = measured_peaks()
    # EM stage = the dominant kernel.  Its time per step comes from CUDA events on the launching stream
    # inside the timed steps (stage 3 brackets the tensor-core launch, the compaction of the buckets it flagged and
    # their re-run on the pair kernel).  Two readings of the same time:
    #  * tensor: dense tcgen05.mma FLOPs the kernel issued (2 M N K per instruction, counted by the library from its
    #    block table) against the measured bf16 GEMM peak -- how busy the tensor pipe is;
    #  * algorithmic: SURVEY 8(d) W_EM lookup-adds (what the reference computes) against the FP32-add peak -- the
    #    figure round 1 reported for the shared-memory kernel, kept for continuity.
    em_launches = args.steps * max(1, -(-(end - begin + 1) // 32768))
    em_ms = stage[3] / max(1, args.steps)
    fp32_peak_tflops = 148 * 128 * sm_max_mhz * 1e6 / 1e12
    algo_tflops = (work / args.steps) / (em_ms * 1e-3) / 1e12 if em_ms > 0 else None
    tensor_tflops = (tensor_flops / args.steps) / (em_ms * 1e-3) / 1e12 if em_ms > 0 and tensor_flops else None
    x = ss.total_lmers(l)
    hb_bytes = (-(-t * cfg["n"] // 4) + 8 * x) * (end - begin + 1)
    hb_ms = (stage[0] + stage[1] + stage[2]) / max(1, args.steps)
    on_tensor = tensor_tflops is not None
    kernel = "em_refine_tc_kernel" if on_tensor else "em_refine_pair_kernel"
    traffic, traffic_src = recorded_traffic(kernel, args.config if not args.trials else None)
    roofline = {
        "bound": "tensor" if on_tensor else "fp32", "kernel": kernel,
        "achieved": tensor_tflops if on_tensor else algo_tflops,
        "peak": bf16_peak if on_tensor else fp32_peak_tflops, "unit": "TFLOP/s",
        "frac": (tensor_tflops / bf16_peak) if on_tensor else ((algo_tflops / fp32_peak_tflops) if algo_tflops else None),
        "traffic": traffic, "traffic_source": traffic_src,
        "launch_ms": em_ms / max(1, em_launches // args.steps),
        "peak_source": (f"MEASURED_PEAKS.json bf16_tflops ({peak_kind}, burst figure: the step lasts about a millisecond)" if on_tensor
                        else f"148 SM x 128 FP32 lanes x {sm_max_mhz:.0f} MHz ({peak_kind} clocks), adds not FMAs"),
        "work": ("dense MMA FLOPs issued: per 128-bucket tile and pass 2*128*columns*K, three bf16 log-odds terms in the E-step "
                 "GEMM (one in the MAX passes), two bf16 responsibility terms in the M-step GEMM" if on_tensor
                 else "SURVEY 8(d) W_EM = sum_b (2 I_b+1) x l + 4 (I_b+1) x FP32 ops (E- and M-step), measured I_b"),
        "algorithmic": {"w_em_tflops": algo_tflops, "fp32_add_peak": fp32_peak_tflops,
                        "frac_of_fp32_add_peak": (algo_tflops / fp32_peak_tflops) if algo_tflops else None,
                        "estep_only_tflops": (lookups / args.steps) / (em_ms * 1e-3) / 1e12 if em_ms > 0 else None,
                        "note": "SURVEY 8(d) W_EM lookup-adds per second against 148 SM x 128 lanes x clock; the one-hot GEMM "
                                "performs these adds on the tensor pipe, so this fraction is not bounded by 1 in principle"},
        "buckets_refined_again": {"pair_kernel": exact_buckets // args.steps, "fp64_kernel": fp64_buckets // args.steps,
                                  "of": result.buckets_enriched},
    }
    if on_tensor:
        # What actually bounds the tensor-core kernel: every pass reads the S block of every tile out of
        # tensor memory, 4 bytes per (bucket, window column), at the measured 64 B/clk/SM of tcgen05.ld.
        W = cfg["n"] - l + 1
        ru = lambda v, m_: -(-v // m_) * m_
        cols = t * ru(ru(-(-W // 2), 16) + ru(W // 2, 16), 32)
        tiles = -(-result.buckets_enriched // 128)
        passes = 5 + 1  # default max_em_iters EM passes + the final E-step
        tmem_bytes = tiles * passes * 128 * cols * 4
        tmem_peak = 148 * 64 * sm_max_mhz * 1e6 / 1e9  # GB/s
        roofline["tmem_read"] = {"achieved": tmem_bytes / (em_ms * 1e-3) / 1e9 if em_ms > 0 else None, "peak": tmem_peak, "unit": "GB/s",
                                 "frac": (tmem_bytes / (em_ms * 1e-3) / 1e9 / tmem_peak) if em_ms > 0 else None,
                                 "note": "S blocks read by tcgen05.ld per step (tiles x 6 passes x 128 rows x padded window columns x 4 B) "
                                         "over the EM stage time, against 148 SMs x 64 B/clk (measured tcgen05.ld rate) x clock"}
    config = workload_config(cfg, m_total, world, args.scaling)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": mean_ms, "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None,
        "dtype": "f32", "data": "synthetic", "config": config,
        "notes": {"trials_per_step_per_gpu": m_per_gpu if args.scaling == "weak" else None,
                  "dtype": "EM sums: bf16 x 3 split operands on tcgen05 with FP32 accumulation (FP32-equivalent); model update FP32; "
                           "decisions within the FP32 error re-run on FP64-assisted kernels; everything else integer",
                  "parallelism": f"trials sharded over {world} GPU(s), one all_gather of the best record",
                  "l2": "256 MiB flush between timed steps (untimed)",
                  "timing": "CUDA events on the launching stream per step, max over ranks"},
        "result": {"consensus": result.consensus.decode(), "score": result.score, "best_trial": result.best_trial,
                   "planted_motif": motif, "recovered": result.consensus.decode() == motif,
                   "buckets_enriched": result.buckets_enriched, "within_d": result.within_d},
        "e2e": {"value": m_total / (mean_e2e * 1e-3), "unit": UNIT, "ms_per_step": mean_e2e,
                "h2d_bytes_per_step": h2d // args.steps, "d2h_bytes_per_step": d2h // args.steps,
                "note": "pm_run_host: pinned host ASCII -> H2D -> encode -> run -> D2H result, every step"},
        "gpu_launches": launches,
        "stage_ms_per_step": {name: stage[i] / args.steps for i, name in
                              enumerate(["keys", "sort", "enrich", "em", "reduce", "score", "upload", "d2h"])},
        "roofline": roofline,
        "roofline_hash_bucket": {"bound": "hbm", "kernels": "hash_bucket_fused (t=20 configs) | project_keys+radix_sort+enrich",
                                 "achieved": (hb_bytes / (hb_ms * 1e-3) / 1e9) if hb_ms > 0 else None, "peak": hbm_peak,
                                 "unit": "GB/s", "frac": (hb_bytes / (hb_ms * 1e-3) / 1e9 / hbm_peak) if hb_ms > 0 else None,
                                 "note": f"algorithmic bytes ceil(t*n/4)+8x per trial; peak {peak_kind}; at t=20 the "
                                         "input is L2-resident so this is a latency/launch-bound stage, see DESIGN.md"},
        "clocks": clocks,
    }

    if not args.no_extras and cfg["t"] <= 100 and world == 1:
        line["time_to_motif"] = time_to_motif(pm, ctx, cfg)
    if ttm_multi is not None:
        line["time_to_motif"] = ttm_multi
    if not args.no_cpu_baseline and world == 1:
        line["cpu_baseline"] = cpu_baseline(cfg)
        if "time_to_motif" in line:
            cpu_time_to_motif(cfg, line["time_to_motif"], line["cpu_baseline"])
    print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


def time_to_motif(pm, ctx, cfg):
    """Wall time from run() entry until the trial T* after which the running best consensus equals
    the planted motif, over several instance seeds, batches of 16 trials."""
    rows = []
    # batch = trials per call.  A 128-bucket tile of the tensor-core EM kernel takes about a millisecond however few
    # tiles there are, so one call over all of C1's 172 trials (138 tiles, one wave of the 148 SMs) costs the same as
    # a call over 32: the whole budget in one batch is the fastest way to the motif.  n = 1000: 64 trials (~285 tiles).
    batch = cfg["m"] if cfg["n"] <= 600 else 64
    for inst_seed in (42, 1, 2, 3, 4):
        bases, offs, motif, _ = pm.generate_planted(cfg["t"], cfg["n"], cfg["l"], cfg["d"], inst_seed)
        ctx.set_sequences(bases, offs)
        t0 = time.perf_counter()
        found_at, first = None, 1
        while first <= cfg["m"] and found_at is None:
            last = min(cfg["m"], first + batch - 1)
            try:
                r = ctx.run(per_trial=False, l=cfg["l"], d=cfg["d"], k=cfg["k"], s=cfg["s"], m=cfg["m"], seed=RUN_SEED,
                            early_stop=0, trial_begin=first, trial_end=last)
                if r["consensus"] == motif:
                    found_at = r["best_trial"]
            except pm.PmError:
                pass
            first = last + 1
        rows.append({"instance_seed": inst_seed, "found": found_at is not None, "t_star": found_at,
                     "ms": 1e3 * (time.perf_counter() - t0)})
    hit = [r for r in rows if r["found"]]
    return {"runs": rows, "ms_median": statistics.median(r["ms"] for r in hit) if hit else None,
            "batch_trials": batch,
            "note": f"wall ms incl. host, batches of {batch} trials, stop at the first batch whose best == planted motif"}


def time_to_motif_sharded(pm, ctx, cfg, dist, rank, world, device, all_gather_merge):
    """time_to_motif on N GPUs.  The planted motif usually appears within the first few trials, so contiguous shards
    would leave every GPU but the first idle: trials are dealt round-robin (trial_stride = N), 16 per rank and round,
    and the ranks exchange their best record after every round (one all_gather of ~300 bytes)."""
    import numpy as np
    import torch
    rows = []
    per_round = 16
    t, l, m = cfg["t"], cfg["l"], cfg["m"]
    for inst_seed in (42, 1, 2, 3, 4):
        bases, offs, motif, _ = pm.generate_planted(t, cfg["n"], l, cfg["d"], inst_seed)
        ctx.set_sequences(bases, offs)
        dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        found_at, base = None, 0
        while base < m and found_at is None:
            begin, end = base + rank + 1, min(m, base + per_round * world)
            out = pm.RunResult()
            pos = np.zeros(t, dtype=np.int32)
            if begin <= end:
                cfg_c = pm.default_config(l=l, d=cfg["d"], k=cfg["k"], s=cfg["s"], m=m, seed=RUN_SEED, early_stop=0,
                                          trial_begin=begin, trial_end=end, trial_stride=world)
                rc = pm.lib().pm_run(ctx._h, C.byref(cfg_c), C.byref(out), pos.ctypes.data_as(C.POINTER(C.c_int32)),
                                     None, None, None, None)
                if rc not in (0, 7):
                    raise pm.PmError(rc, pm.lib().pm_last_error().decode())
            try:
                merged, _ = all_gather_merge(out, pos, t, l, False, device=device)
                if merged.consensus.decode() == motif:
                    found_at = int(merged.best_trial)
            except pm.PmError:
                pass  # no rank enriched a bucket in this round
            base += per_round * world
        torch.cuda.synchronize()
        rows.append({"instance_seed": inst_seed, "found": found_at is not None, "t_star": found_at,
                     "ms": 1e3 * (time.perf_counter() - t0)})
    hit = [r for r in rows if r["found"]]
    return {"runs": rows, "ms_median": statistics.median(r["ms"] for r in hit) if hit else None, "n_gpus": world,
            "note": f"wall ms incl. host on rank 0; round-robin shards over {world} GPUs, rounds of {per_round} trials per GPU, "
                    "one all_gather per round; stop at the first round whose merged best == planted motif"}


def cpu_time_to_motif(cfg, ttm, baseline):
    """The reference's time to the same trial T*: projmotif::run over trials 1..T* (workers = host cores, its
    blocks of `workers` trials run to completion, driver.hpp:186-209) on the instances time_to_motif() solved."""
    oracle, kind = load_cpu_oracle()
    if kind != "reference":
        return
    cores = os.cpu_count() or 1
    rows = []
    for r in ttm["runs"]:
        if not r["found"]:
            continue
        ss, motif, _ = oracle.generate_planted(cfg["t"], cfg["n"], cfg["l"], cfg["d"], r["instance_seed"])
        t0 = time.perf_counter()
        got = oracle.run(ss, l=cfg["l"], d=cfg["d"], k=cfg["k"], s=cfg["s"], m=r["t_star"], seed=RUN_SEED, early_stop=0,
                         workers=cores)
        r["cpu_ms"] = 1e3 * (time.perf_counter() - t0)
        r["cpu_found"] = got["consensus"] == motif
        rows.append(r["cpu_ms"])
    if rows:
        ttm["cpu_ms_median"] = statistics.median(rows)
        ttm["cpu_note"] = f"projmotif::run(m = T*, workers={cores}) wall ms on the same instances ({baseline['kind']})"


def cpu_baseline(cfg):
    oracle, kind = load_cpu_oracle()
    ss, _, _ = oracle.generate_planted(cfg["t"], cfg["n"], cfg["l"], cfg["d"], INSTANCE_SEED)
    cores = os.cpu_count() or 1
    workers = cores if kind == "reference" else 1
    if cfg.get("extrapolate_cpu"):
        value, info = cpu_extrapolated_trials_per_second(oracle, ss, cfg, cores)
        return {"value": value, "unit": UNIT, "cores": cores, "kind": kind, "sample": f"EXTRAPOLATED from {info}"}
    # calibrate on `workers` trials, then size the sample for ~15 s of wall time
    rate, dt = cpu_trials_per_second(oracle, kind, ss, cfg, max(workers, 2), workers)
    sample = int(max(workers, rate * 15.0))  # ~15 s; trials are i.i.d. in cost, so the sample may exceed m
    sample = max(workers, (sample // workers) * workers)
    value, dt = cpu_trials_per_second(oracle, kind, ss, cfg, sample, workers)
    return {"value": value, "unit": UNIT, "cores": workers, "kind": kind,
            "sample": f"{sample} of the workload's trials through projmotif::run (reference headers, -O3 -DNDEBUG, "
                      f"workers={workers}) in {dt:.1f} s on {cores} host cores"}


def main():
    args = parse_args()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        run_reference_arm(args, cfg, rank, world)
    else:
        run_b200_arm(args, cfg, rank, world, local_rank)


if __name__ == "__main__":
    main()
