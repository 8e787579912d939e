python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
run() { python bench.py --steps 40 --warmup 5 --no-fit --no-cpu-baseline --no-extras --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$1', 'value', round(d['value']/1e9,3), 'kernel_ms', round(r['kernel_ms'],4), 'frac', round(r['frac'],4))"; }
run base; run base2
rm -f paper_2512_11624_b200/_lib/obj/train_planar.o; make -s -C paper_2512_11624_b200/csrc EXTRA=-DGSVR_NO_REFINE >/dev/null 2>&1; run norefine; run norefine2
rm -f paper_2512_11624_b200/_lib/obj/train_planar.o; make -s -C paper_2512_11624_b200/csrc >/dev/null 2>&1
