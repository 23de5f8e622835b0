#!/bin/bash
# Round profile recipe (run under gpurun from the repo root): GPU tests, bench
# lines for c1/c2/c3/c5, the c2 launch list, and ncu --set full of the top kernels.
set -u
mkdir -p gpurun_out
O=gpurun_out
python bench.py > $O/bench_c2.json 2> $O/bench_c2.err
python bench.py --config c1 > $O/bench_c1.json 2> $O/bench_c1.err
python bench.py --config c3 --steps 3 --no-cpu-baseline > $O/bench_c3.json 2> $O/bench_c3.err
python bench.py --config c5 --steps 3 --no-cpu-baseline > $O/bench_c5.json 2> $O/bench_c5.err
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1"
$CMD > $O/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c2.csv $CMD > $O/ncu_launch.log 2>&1
$CMD > $O/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:'k_vix_quads|k_viewshed_evk|k_site_loop' -s 0 -c 3 -o $O/prof_c2 $CMD > $O/ncu_full2.log 2>&1
python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --sharded > $O/bench_c2_sharded1.json 2> $O/bench_c2_sharded1.err
python bench.py --config c4 --steps 2 --warmup 3 --no-cpu-baseline > $O/bench_c4.json 2> $O/bench_c4.err
python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo rc=$? >> $O/pytest_gpu.log
echo done
