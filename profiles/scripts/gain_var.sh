#!/bin/bash
# SITE gain-pass variants (build/var/libtxsite_$v.so via build_variant.sh): kernel-level TB/s per config
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
O=gpurun_out/gain_var.log; : > $O
for v in default ${VARS}; do
  if [ $v = default ]; then unset TXS_LIB; else export TXS_LIB=$PWD/build/var/libtxsite_$v.so; fi
  for c in ${CFGS:-c2 c3 c5}; do python profiles/scripts/gain_once.py $c 2>&1 | tail -1 | sed "s/^/$v $c /" >> $O; done
done
