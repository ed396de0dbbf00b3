"""Writes profiles/r2_sass_evidence.txt: per kernel of the in-tree libpm_b200.so, the Blackwell-specific SASS mnemonics
it contains (tcgen05 = UTCHMMA / LDTM / STTM / UTCBAR, TMA bulk copies = UBLKCP, mbarriers = SYNCS, setmaxnreg =
USETMAXREG, packed FP32x2 = FADD2 / FMUL2 / FFMA2, global reductions = REDG / ATOMG) with one sample line each.
    python tools/sass_evidence.py            (needs cuobjdump; no GPU)"""
import collections
import os
import re
import subprocess

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(REPO, "paper_1605_06904_b200", "libpm_b200.so")
WANT = ["em_refine_tc_kernelILi16", "em_refine_pair_kernelILi8", "em_refine_f64_kernel", "hash_bucket_fused_kernel", "plan_sample_kernel", "trial_reduce_kernel",
        "count_hist_kernel", "count_scan_kernel", "count_scatter_kernel", "count_order_kernel", "encode_kernel",
        "hamming_scan_kernel", "median_string_kernel", "mt64_stream_kernel",
        "radix_scatter_kernelIjLb0", "project_keys_kernelIj"]
PAT = re.compile(r"\b(UTCHMMA|LDTM|STTM|UTCBAR|UBLKCP|SYNCS|USETMAXREG|FADD2|FMUL2|FFMA2|REDG|ATOMG|ATOMS|REDUX|MUFU\.EX2|F2FP|"
                 r"POPC|MATCH|ELECT|DADD|DFMA)\b")
SHOW = ("UTCHMMA", "LDTM", "STTM", "UTCBAR", "USETMAXREG", "UBLKCP", "SYNCS", "FADD2", "FFMA2", "REDG", "ATOMG", "DFMA", "POPC", "MATCH")


def main():
    sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
    size = os.path.getsize(LIB)
    funcs = re.split(r"\n\s*Function : ", sass)
    out = [f"SASS evidence: {os.path.relpath(LIB, REPO)} ({size / 1e6:.1f} MB, {len(funcs) - 1} sm_100a kernels), `cuobjdump -sass`.",
           "Per kernel: instruction count, the architecture-specific mnemonics it contains (count), one sample line each.",
           "  UTCHMMA = tcgen05.mma kind::f16 | LDTM / STTM = tcgen05.ld / st | UTCBAR = tcgen05.commit | UBLKCP = cp.async.bulk (TMA)",
           "  SYNCS = mbarrier | USETMAXREG = setmaxnreg | FADD2 / FMUL2 / FFMA2 = packed FP32x2 | REDG / ATOMG = global reductions", ""]
    for f in funcs[1:]:
        name = f.split("\n", 1)[0].strip()
        if not any(w in name for w in WANT):
            continue
        dem = subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip().replace("(anonymous namespace)", "{anonymous}").split("(")[0]
        lines = [ln for ln in f.split("\n") if re.search(r"/\*[0-9a-f]{4,}\*/", ln) and not re.match(r"\s*/\* 0x", ln)]
        cnt, sample = collections.Counter(), {}
        for ln in lines:
            m = PAT.search(ln)
            if m:
                cnt[m.group(1)] += 1
                sample.setdefault(m.group(1), re.sub(r"\s+", " ", re.sub(r"/\*.*?\*/", "", ln)).strip())
        out.append(f"== {dem}: {len(lines)} instructions")
        out.append("   " + ", ".join(f"{k} x{v}" for k, v in sorted(cnt.items(), key=lambda kv: -kv[1])))
        out += [f"     {sample[k]}" for k in SHOW if k in sample]
        out.append("")
    with open(os.path.join(REPO, "profiles", "r2_sass_evidence.txt"), "w") as fh:
        fh.write("\n".join(out))
    print("\n".join(out))


if __name__ == "__main__":
    main()
