python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1
run() { python bench.py --steps 30 --warmup 5 --no-fit --no-cpu-baseline --no-extras --e2e-steps 1 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$1', 'value', round(d['value']/1e9,3), 'kernel_ms', round(r['kernel_ms'],4), 'frac', round(r['frac'],4))"; }
run base
for u in 2 4; do rm -f paper_2512_11624_b200/_lib/obj/train_planar.o; make -s -C paper_2512_11624_b200/csrc EXTRA=-DGSVR_FWD_UNROLL=$u >/dev/null 2>&1; run unroll$u; done
