mkdir -p gpurun_out
O=gpurun_out/var.log; : > $O
for v in base k8 k16; do
  if [ $v = base ]; then unset TXS_LIB; else export TXS_LIB=$PWD/build/var/libtxsite_$v.so; fi
  python profiles/scripts/stage_time.py c4 vix 1 2>&1 | tail -1 | sed "s/^/$v /" >> $O
  python profiles/scripts/stage_time.py c1 vix 3 2>&1 | tail -1 | sed "s/^/$v /" >> $O
done
