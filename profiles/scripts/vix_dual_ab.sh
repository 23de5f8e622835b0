#!/bin/bash
# k_vix_lanes group size chosen per launch by k_vix_sample (TXS_VIX_DUAL=1, default) against 16-step groups only:
# sampled failing fractions per config and the VIX kernel / step times.   usage: vix_dual_ab.sh "c3 c4 c1"
O=gpurun_out; mkdir -p $O
for c in $1; do
  TXS_VIX_VERBOSE=1 python profiles/scripts/vix_once.py $c 2>&1 | grep "VIX rows" | head -3
done
profiles/scripts/vix_env_ab.sh "$1" TXS_VIX_DUAL "0 1"; cat $O/envab.txt
