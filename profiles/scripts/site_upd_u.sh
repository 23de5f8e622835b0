mkdir -p gpurun_out
O=gpurun_out/var.log; : > $O
for v in base u8 u2; do
  if [ $v = base ]; then unset TXS_LIB; else export TXS_LIB=$PWD/build/var/libtxsite_$v.so; fi
  for c in c2 c3 c5; do python profiles/scripts/stage_time.py $c site 1 2>&1 | tail -1 | sed "s/^/$v /" >> $O; done
done
