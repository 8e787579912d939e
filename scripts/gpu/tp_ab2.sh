python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
python -m pytest tests/test_gpu_l1.py tests/test_gpu_parity.py tests/test_gpu_fit.py -x -q 2>&1 | tail -2
run() { python bench.py --steps 40 --warmup 5 --no-fit --no-cpu-baseline --no-extras --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$1', 'value', round(d['value']/1e9,3), 'kernel_ms', round(r['kernel_ms'],4), 'frac', round(r['frac'],4))"; }
run new; run new2
