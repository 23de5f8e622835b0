# A/B of VIX builds (build_variant.sh): parity subset + c2/c3 stage times
mkdir -p gpurun_out
O=gpurun_out/var.log; : > $O
for v in base ${VARIANTS}; do
  if [ $v = base ]; then unset TXS_LIB; else export TXS_LIB=$PWD/build/var/libtxsite_$v.so; fi
  python -m pytest tests -m gpu -x -q -k "vix_paths or vix_rows" 2>&1 | tail -1 | sed "s/^/$v test: /" >> $O
  for c in ${CFGS:-c2 c3}; do python profiles/scripts/stage_time.py $c vix 2 2>&1 | tail -1 | sed "s/^/$v /" >> $O; done
done
