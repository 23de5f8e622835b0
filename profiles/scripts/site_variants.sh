# A/B of SITE gain-pass builds (build_variant.sh ... site): parity subset + mode-1 round streaming
mkdir -p gpurun_out
O=gpurun_out/var.log; : > $O
for v in base ${VARIANTS}; do
  if [ $v = base ]; then unset TXS_LIB; else export TXS_LIB=$PWD/build/var/libtxsite_$v.so; fi
  python -m pytest tests -m gpu -x -q -k "site or gain or marginal" 2>&1 | tail -1 | sed "s/^/$v test: /" >> $O
  for c in c2 c3 c5; do
    TXS_GAIN_REG=1 python profiles/scripts/stage_time.py $c site1 2 2>&1 | tail -1 | sed "s/^/$v /" >> $O
  done
done
