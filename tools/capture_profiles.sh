#!/bin/bash
# Run on the GPU box (under gpurun): bench records of every BASELINE configuration, the reference arm, ncu launch
# lists and `--set full` captures of the dominant kernels.  Everything lands in gpurun_out/r2_*; tools/refresh_records.py
# then copies the records and text summaries into profiles/.  Numbers printed under ncu are never bench values.
set -u
OUT=gpurun_out
mkdir -p $OUT
B="timeout 900 python bench.py"
$B --steps 20 --warmup 5 > $OUT/r2_bench_c1.json 2> $OUT/r2_bench_c1.err
for c in c2 c3 c3b c4; do $B --config $c --steps 5 --warmup 3 > $OUT/r2_bench_$c.json 2> $OUT/r2_bench_$c.err; done
$B --config c5 --steps 3 --warmup 3 > $OUT/r2_bench_c5.json 2> $OUT/r2_bench_c5.err
$B --config c5b --steps 2 --warmup 3 > $OUT/r2_bench_c5b.json 2> $OUT/r2_bench_c5b.err
$B --impl reference --steps 3 --warmup 1 > $OUT/r2_bench_c1_reference_arm.json 2> $OUT/r2_bench_c1_reference_arm.err
$B --scaling strong --config c4 --steps 3 --warmup 3 --no-cpu-baseline --no-extras > $OUT/r2_bench_c4_strong_n1.json 2>/dev/null
# launch lists (shares of the step, cold-cache and serialised)
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/r2_launches_c1.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-extras > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/r2_launches_c2.csv \
    python bench.py --config c2 --steps 1 --warmup 1 --no-cpu-baseline --no-extras > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file $OUT/r2_launches_c5.csv \
    python bench.py --config c5 --steps 1 --warmup 1 --no-cpu-baseline --no-extras > /dev/null 2>&1
# full captures: the tensor-core EM kernel on C1 and C2, the pair kernel (flagged re-run) on C2, the counting-sort
# kernels and the radix-sort kernels on C5
timeout 600 ncu --set full --clock-control none --import-source on -k regex:em_refine_tc -c 1 -s 2 -o $OUT/r2_em_refine_tc_c1 \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-extras > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:em_refine_tc -c 1 -s 1 -o $OUT/r2_em_refine_tc_c2 \
    python bench.py --config c2 --steps 1 --warmup 1 --no-cpu-baseline --no-extras > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none -k regex:"count_|hash_bucket_fused" -c 6 -s 6 -o $OUT/r2_count_c5 \
    python bench.py --config c5 --steps 1 --warmup 1 --no-cpu-baseline --no-extras > /dev/null 2>&1
PM_B200_COUNT_HASH=0 timeout 600 ncu --set full --clock-control none -k regex:"project_keys|radix_|enrich_kernel" -c 12 -s 12 -o $OUT/r2_sort_c5 \
    python bench.py --config c5 --steps 1 --warmup 1 --no-cpu-baseline --no-extras > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none -k regex:hash_bucket_fused -c 1 -s 2 -o $OUT/r2_hash_fused_c1 \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-extras > /dev/null 2>&1
# digest on the box: the reports are too large to bring back (gpurun returns at most 64 MiB)
PM_PROFILES_DST=$OUT/profiles_r2 python tools/refresh_records.py > $OUT/r2_refresh.log 2>&1
rm -f $OUT/r2_em_refine_tc_c2.ncu-rep $OUT/r2_count_c5.ncu-rep $OUT/r2_sort_c5.ncu-rep $OUT/r2_hash_fused_c1.ncu-rep
ls -la $OUT $OUT/profiles_r2 | tail -40
