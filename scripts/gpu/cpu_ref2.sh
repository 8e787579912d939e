python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
SKIP_CFG1=1 CFG2_REFRESHES=58 timeout 1800 python scripts/cpu_reference_host.py > gpurun_out/cpu_ref2.log 2>&1
run() { python bench.py --steps 30 --warmup 5 --no-fit --no-cpu-baseline --no-extras --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$1', round(d['value']/1e9,3), 'kernel_ms', round(r['kernel_ms'],4), 'frac', round(r['frac'],4))"; }
run base
rm -f paper_2512_11624_b200/_lib/obj/train_planar.o; make -s -C paper_2512_11624_b200/csrc EXTRA=-DGSVR_PLANAR_MINB=4 >/dev/null 2>&1
grep -A3 "ILb1" paper_2512_11624_b200/_lib/obj/train_planar.ptxas.log | grep -i "regis\|spill"
run minb4_smem
python - <<'PY'
import sys; sys.path.insert(0,'.')
from paper_2512_11624_b200._native import lib
PY
rm -f paper_2512_11624_b200/_lib/obj/train_planar.o; make -s -C paper_2512_11624_b200/csrc >/dev/null 2>&1
