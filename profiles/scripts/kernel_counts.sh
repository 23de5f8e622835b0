#!/bin/bash
# Per-config counters of the main kernels (run under gpurun from the repo root):
# each config's one_run.py exits 0 without ncu first, then runs under ncu with
# the counters bench.py's roofline needs; counts_summary.py turns the CSVs into
# profiles/kernel_counts.json.   usage: kernel_counts.sh c1 c2 c3 c4 c5
set -u
O=gpurun_out
mkdir -p $O
M=gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_write.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__throughput.avg.pct_of_peak_sustained_elapsed
K='regex:k_batch_|k_vix_lanes|k_vix_quads|k_vix<|k_viewshed_evk|k_viewshed_ev<|k_viewshed<|k_gain_full|k_gain_tiled|k_site_loop|k_findmax|k_vix_fp64_ties|k_vs_fp64_ties'
for c in "$@"; do
  python profiles/scripts/one_run.py --config $c > $O/one_$c.log 2>&1 && \
  ncu --metrics $M --clock-control none -k "$K" --csv --log-file $O/counts_$c.csv \
      python profiles/scripts/one_run.py --config $c > $O/ncu_counts_$c.log 2>&1
  echo "$c rc=$?" >> $O/counts_rc.txt
done
