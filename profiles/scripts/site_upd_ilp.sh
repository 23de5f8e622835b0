mkdir -p gpurun_out
O=gpurun_out/var.log; : > $O
python -m pytest tests -m gpu -x -q -k "site or shard" 2>&1 | tail -1 | sed "s/^/test: /" >> $O
for c in c1 c2 c3 c5; do python profiles/scripts/stage_time.py $c site 2 2>&1 | tail -1 >> $O; done
