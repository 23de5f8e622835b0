mkdir -p gpurun_out
O=gpurun_out/var.log; : > $O
for v in base vs480x3; do
  if [ $v = base ]; then unset TXS_LIB; else export TXS_LIB=$PWD/build/var/libtxsite_$v.so; fi
  python -m pytest tests -m gpu -x -q -k "k_paths" 2>&1 | tail -1 | sed "s/^/$v test: /" >> $O
  python profiles/scripts/stage_time.py c5 viewshed 1 2>&1 | tail -1 | sed "s/^/$v /" >> $O
done
