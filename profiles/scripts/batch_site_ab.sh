set -x
export TXS_SITE_BATCH_VERBOSE=1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "site or pipeline or smoke" 2>&1 | tail -15
for c in c1 c2 c3 c5; do
 timeout 600 python bench.py --config $c --steps 3 --warmup 1 --no-cpu-baseline > gpurun_out/batch_$c.log 2>gpurun_out/batch_$c.err; echo "$c rc=$?"; grep -h "batched SITE" gpurun_out/batch_$c.err | tail -1
 TXS_SITE_BATCH=0 timeout 600 python bench.py --config $c --steps 3 --warmup 1 --no-cpu-baseline > gpurun_out/serial_$c.log 2>&1
done
python - <<'PY'
import json
for c in ['c1','c2','c3','c5']:
    for k in ['batch','serial']:
        try:
            l=[x for x in open(f'gpurun_out/{k}_{c}.log') if x.startswith('{')][-1]
            j=json.loads(l); print(c,k,j['value'],j.get('stages'))
        except Exception as e: print(c,k,'ERR',e)
PY
