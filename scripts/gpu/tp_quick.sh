python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
python -m pytest tests/test_gpu_parity.py tests/test_gpu_l1.py tests/test_gpu_fit.py -x -q 2>&1 | tail -3
python bench.py --steps 30 --warmup 5 --no-fit --no-cpu-baseline --no-extras --e2e-steps 1 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('value', d['value']/1e9, 'kernel_ms', r['kernel_ms'], 'frac', r['frac'], 'pass_ms', r['train_pass_ms'])"
