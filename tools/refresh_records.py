"""Copies the round-2 records of tools/capture_profiles.sh from gpurun_out/ into profiles/, writes the text summaries
(launch shares, ncu --set full digests, traffic.json) and rewrites the measured tables of DESIGN.md / README.md from
them, so that the documented numbers are the recorded ones.

    python tools/refresh_records.py            (after `gpurun -- bash tools/capture_profiles.sh`)
"""
import collections
import csv
import json
import os
import re
import shutil
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
os.chdir(REPO)
SRC = "gpurun_out"
DST = os.environ.get("PM_PROFILES_DST", "profiles")  # on the GPU box: a directory under gpurun_out/ (only that comes back)
CONFIGS = ("c1", "c2", "c3", "c3b", "c4", "c5", "c5b")
NAMES = {"c1": "C1 (15,4) t=20 n=600, m=172", "c2": "C2 (16,5) t=20 n=1000, m=1293", "c3": "C3 (18,6), m=2218",
         "c3b": "C3b (19,6), m=711", "c4": "C4 (20,7), m=3421", "c5": "C5 (15,4) t=10,000 n=1000, k=10 s=19, m=2",
         "c5b": "C5b same set, k=7 s=4, m=1"}


def last_json(path):
    with open(path) as f:
        return json.loads(f.read().strip().splitlines()[-1])


def launch_shares(csv_path, out_path, title):
    rows = [r for r in csv.reader(open(csv_path)) if len(r) > 5]
    hdr, data = None, []
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
        elif hdr and len(r) == len(hdr):
            data.append(r)
    ik, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0.0, 0])
    for r in data:
        v, u = float(r[iv].replace(",", "")), r[iu]
        us = v / 1000 if u in ("ns", "nsecond") else v if u in ("us", "usecond") else v * 1000
        name = re.sub(r"\(.*", "", r[ik]).strip()
        agg[name][0] += us
        agg[name][1] += 1
    tot = sum(v[0] for v in agg.values())
    out = [title, "per-launch times are cold-cache and serialised: compare SHARES, not absolutes "
                  "(the at::...FillFunctor launches are bench.py's untimed L2 flush)", ""]
    for k, (us, n) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
        out.append(f"{us:12.1f} us {n:4d}x {100 * us / tot:5.1f}%  {k}")
    open(out_path, "w").write("\n".join(out) + "\n")


def main():
    os.makedirs(DST, exist_ok=True)
    rec = {}
    for c in CONFIGS:
        src = f"{SRC}/r2_bench_{c}.json"
        if os.path.exists(src) and os.path.getsize(src) > 0:
            shutil.copy(src, f"{DST}/r2_bench_{c}.json")
        if os.path.exists(f"{DST}/r2_bench_{c}.json"):
            rec[c] = last_json(f"{DST}/r2_bench_{c}.json")
    for extra in ("r2_bench_c1_reference_arm.json", "r2_bench_c4_strong_n1.json"):
        if os.path.exists(f"{SRC}/{extra}") and os.path.getsize(f"{SRC}/{extra}") > 0:
            shutil.copy(f"{SRC}/{extra}", f"{DST}/{extra}")
    for c, cmd in (("c1", "python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-extras (C1, 172 trials/step)"),
                   ("c2", "python bench.py --config c2 --steps 1 --warmup 1 ... (C2, 1,293 trials/step)"),
                   ("c5", "python bench.py --config c5 --steps 1 --warmup 1 ... (C5, 2 trials/step)")):
        p = f"{SRC}/r2_launches_{c}.csv"
        if os.path.exists(p):
            shutil.copy(p, f"{DST}/r2_launches_{c}.csv")
            launch_shares(p, f"{DST}/r2_launch_shares_{c}.txt",
                          f"ncu --metrics gpu__time_duration.sum --clock-control none: {cmd}")
    # ncu --set full digests + traffic.json
    pairs = []
    for rep, cfg in (("r2_em_refine_tc_c1", "c1"), ("r2_em_refine_tc_c2", "c2"), ("r2_count_c5", "c5"), ("r2_sort_c5", "c5"),
                     ("r2_hash_fused_c1", "c1")):
        path = f"{SRC}/{rep}.ncu-rep"
        if not os.path.exists(path):
            continue
        args = [sys.executable, "tools/ncu_summary.py", path] + (["0.012"] if "em_refine" in rep else [])
        txt = subprocess.run(args, capture_output=True, text=True).stdout
        open(f"{DST}/{rep}_ncu_full.txt", "w").write(
            f"ncu --set full --clock-control none (tools/capture_profiles.sh), digest by tools/ncu_summary.py of {rep}.ncu-rep\n\n" + txt)
        pairs += [cfg, path]
    if os.path.isdir(f"{SRC}/profiles_r2") and DST != f"{SRC}/profiles_r2":
        # digests made on the GPU box (most reports are too large to bring back): they are the record
        for name in sorted(os.listdir(f"{SRC}/profiles_r2")):
            if name.endswith("_ncu_full.txt") or name == "traffic.json":
                shutil.copy(f"{SRC}/profiles_r2/{name}", f"{DST}/{name}")
    elif pairs:
        if os.path.exists(f"{DST}/traffic.json"):
            os.remove(f"{DST}/traffic.json")
        subprocess.run([sys.executable, "tools/ncu_traffic.py"] + pairs, check=True, stdout=subprocess.DEVNULL,
                       env=dict(os.environ, PM_PROFILES_DST=DST))

    fmt = lambda x: f"{x / 1000:.1f} k" if x >= 1000 else f"{x:.2f}"
    rows = ["| config | trials/s (HBM-resident) | e2e trials/s | EM share of step | roofline kernel | achieved / peak | frac | "
            "buckets re-run (pair / FP64) of | reference CPU on the box (16 cores), trials/s |", "|---|---|---|---|---|---|---|---|---|"]
    for c in CONFIGS:
        if c not in rec:
            continue
        d = rec[c]
        rf = d["roofline"]
        share = 100 * d["stage_ms_per_step"]["em"] / d["ms_per_step"]
        again = rf.get("buckets_refined_again", {})
        cpu = d.get("cpu_baseline", {}).get("value")
        rows.append(f"| {NAMES[c]} | {fmt(d['value'])} | {fmt(d['e2e']['value'])} | {share:.1f} % | `{rf['kernel'].replace('_kernel', '')}` ({rf['bound']}) | "
                    f"{rf['achieved']:.1f} / {rf['peak']:.1f} {rf['unit']} | {rf['frac']:.3f} | {again.get('pair_kernel', 0)} / {again.get('fp64_kernel', 0)} of "
                    f"{again.get('of', 0)} | {('%.4g' % cpu) if cpu else 'n/a'}{' (extrapolated)' if c.startswith('c5') and cpu else ''} |")
    table = "\n".join(rows)
    s = open("DESIGN.md").read()
    a, b = s.index("<!-- r2-table-begin -->"), s.index("<!-- r2-table-end -->")
    s = s[:a] + "<!-- r2-table-begin -->\n" + table + "\n" + s[b:]
    if "c1" in rec and "time_to_motif" in rec["c1"]:
        ttm = rec["c1"]["time_to_motif"]
        s = re.sub(r"<!-- r2-ttm -->.*?for the reference\.(?:[0-9. a-z]*for the reference\.)*", f"<!-- r2-ttm -->median {ttm['ms_median']:.2f} ms against {ttm.get('cpu_ms_median', 0):.0f} ms for the reference.", s)
    open("DESIGN.md", "w").write(s)
    print(table)


if __name__ == "__main__":
    main()
