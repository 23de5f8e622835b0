# SITE graph-path launch parameters on c5 (neighbour update threads / grid, argmax grid)
mkdir -p gpurun_out
O=gpurun_out/var.log; : > $O
for v in base u64 u256; do
  if [ $v = base ]; then unset TXS_LIB; else export TXS_LIB=$PWD/build/var/libtxsite_$v.so; fi
  for m in 4 8 16; do TXS_UPD_MULT=$m python profiles/scripts/stage_time.py c5 site 1 2>&1 | tail -1 | sed "s/^/$v upd=$m /" >> $O; done
done
unset TXS_LIB
for m in 1 4 8; do TXS_ARGMAX_MULT=$m python profiles/scripts/stage_time.py c5 site 1 2>&1 | tail -1 | sed "s/^/argmax=$m /" >> $O; done
