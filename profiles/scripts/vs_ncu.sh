#!/bin/bash
# ncu --set full (+ source) of the VIEWSHED sweep kernel per config, and the per-kernel times of the
# batched SITE rounds: vs_ncu.sh c3 c5
set -u
O=gpurun_out; mkdir -p $O
for c in "$@"; do
  python profiles/scripts/vs_once.py $c > $O/vs_once_$c.log 2>&1 && \
  timeout 1200 ncu --set full --import-source on --clock-control none -k regex:k_viewshed_evk -c 1 -o $O/r02_vs_$c -f \
      python profiles/scripts/vs_once.py $c > $O/ncu_vs_$c.log 2>&1
  python profiles/scripts/ncu_summary.py $O/r02_vs_$c.ncu-rep > $O/r02_vs_$c.csv
  python profiles/scripts/one_run.py --config $c > $O/one_$c.log 2>&1 && \
  timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_batch --csv --log-file $O/batch_launches_$c.csv \
      python profiles/scripts/one_run.py --config $c > $O/ncu_batch_$c.log 2>&1
done
