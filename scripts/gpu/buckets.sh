timeout 900 python -m pytest tests/test_gpu_buckets.py tests/test_gpu_parity.py -q -p no:cacheprovider > gpurun_out/buckets_tests.log 2>&1
run() { GSVR_TILE_BUCKETS=$2 timeout 900 python bench.py --config $3 --steps 30 --warmup 5 --no-fit --no-cpu-baseline --no-extras --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$1 $3', round(d['value']/1e9,4), 'kernel_ms', round(r['kernel_ms'],4), 'frac', round(r['frac'],4))"; }
for c in cfg2 cfg4; do run on 1 $c; run off 0 $c; done > gpurun_out/buckets.log 2>&1
