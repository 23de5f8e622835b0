mkdir -p gpurun_out
O=gpurun_out/var.log; : > $O
for v in k8 k16; do
  export TXS_LIB=$PWD/build/var/libtxsite_$v.so
  python -m pytest tests -m gpu -x -q -k "vix_paths or vix_rows" 2>&1 | tail -1 | sed "s/^/$v test: /" >> $O
  for st in 0 8 16 32; do
    if [ $st = 0 ]; then unset TXS_VIX_STRIP; else export TXS_VIX_STRIP=$st; fi
    python profiles/scripts/stage_time.py c2 vix 2 2>&1 | tail -1 | sed "s/^/$v strip=$st /" >> $O
  done
  unset TXS_VIX_STRIP
  python profiles/scripts/stage_time.py c3 vix 2 2>&1 | tail -1 | sed "s/^/$v /" >> $O
done
