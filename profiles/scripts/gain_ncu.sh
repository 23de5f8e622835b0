#!/bin/bash
# ncu --set full of one streaming gain pass per layout (cum-aligned rows / 8x8 tiles): gain_ncu.sh c4 [c3 ...]
cd "$(dirname "$0")/../.."
O=gpurun_out; mkdir -p $O
for c in "$@"; do
  for k in full t8; do
    TXS_GAIN_PASS=$k timeout 900 ncu --set full --import-source on --clock-control none --cache-control none \
      -k regex:k_gain_full -s 3 -c 1 -o $O/gain_${c}_$k -f python profiles/scripts/gain_once.py $c > $O/gain_ncu_${c}_$k.log 2>&1
    python profiles/scripts/ncu_summary.py $O/gain_${c}_$k.ncu-rep > $O/gain_${c}_$k.csv
  done
done
