mkdir -p gpurun_out
O=gpurun_out/var.log; : > $O
python -m pytest tests -m gpu -x -q -k "vix" 2>&1 | tail -1 | sed "s/^/test: /" >> $O
for c in c1 c2 c3; do for v in 0 1; do TXS_VIX_CS=$v python profiles/scripts/stage_time.py $c vix 2 2>&1 | tail -1 | sed "s/^/cs=$v /" >> $O; done; done
