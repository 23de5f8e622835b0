mkdir -p gpurun_out
O=gpurun_out/var.log; : > $O
for v in k8 k4 k8t256; do
  export TXS_LIB=$PWD/build/var/libtxsite_$v.so
  python -m pytest tests -m gpu -x -q -k "vix_paths or vix_rows" 2>&1 | tail -1 | sed "s/^/$v test: /" >> $O
  for c in c1 c2 c3; do python profiles/scripts/stage_time.py $c vix 2 2>&1 | tail -1 | sed "s/^/$v /" >> $O; done
done
