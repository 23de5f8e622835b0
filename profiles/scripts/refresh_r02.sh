#!/bin/bash
# Round-2 evidence refresh (run under gpurun from the repo root): per-config ncu
# counters, the c3 launch list, one ncu --set full capture of the top VIX
# kernel at c3, the five bench lines and the reference arm at c3.
set -u
O=gpurun_out; mkdir -p $O
profiles/scripts/kernel_counts.sh c1 c2 c3 c4 c5
python profiles/scripts/counts_summary.py c1 c2 c3 c4 c5 > $O/counts_summary.log 2>&1   # the bench lines below read it
python bench.py --config c3 --steps 2 --warmup 1 --no-cpu-baseline > $O/ll_pre.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file $O/launches_c3.csv \
    python bench.py --config c3 --steps 2 --warmup 1 --no-cpu-baseline > $O/ll_ncu.log 2>&1
python profiles/scripts/vix_once.py c3 > $O/vix_once.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:k_vix_lanes -c 1 -o $O/r02_vix_c3 -f \
    python profiles/scripts/vix_once.py c3 > $O/ncu_vix_full.log 2>&1
profiles/scripts/gain_ncu.sh c3 c4
for c in c3 c1 c2 c4 c5; do timeout 900 python bench.py --config $c > $O/final_bench_$c.log 2>&1; done
timeout 900 python bench.py --impl reference > $O/final_ref_c3.log 2>&1
echo done > $O/refresh_done.txt
