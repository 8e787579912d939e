python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
python -m pytest tests/test_gpu_parity.py -q -k "global_memory or backward_matches" 2>&1 | tail -2
python bench.py --steps 30 --warmup 5 --no-fit --no-cpu-baseline --no-extras --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('cfg2', round(d['value']/1e9,3), 'kernel_ms', round(r['kernel_ms'],4), 'frac', round(r['frac'],4))"
for v in 1 0; do GSVR_BREC_GLOBAL=$v python bench.py --config cfg4 --steps 10 --warmup 3 --no-fit --no-cpu-baseline --no-extras --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('cfg4 bglob=$v', round(d['value']/1e9,3), 'kernel_ms', round(r['kernel_ms'],4), 'frac', round(r['frac'],4))"; done
