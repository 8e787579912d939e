run() { python bench.py --steps 50 --warmup 5 --no-fit --no-cpu-baseline --no-extras --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$1', round(d['value']/1e9,4), 'kernel_ms', round(r['kernel_ms'],4), 'frac', round(r['frac'],4))"; }
cp -r paper_2512_11624_b200/csrc /tmp/csrc_new
git stash -q 2>/dev/null || true
for i in 1 2; do run new; done
git checkout -q HEAD~1 -- paper_2512_11624_b200/csrc/train_planar.cu paper_2512_11624_b200/csrc/batch.cu paper_2512_11624_b200/csrc/batch.cuh
rm -f paper_2512_11624_b200/_lib/obj/*.o; make -s -C paper_2512_11624_b200/csrc >/dev/null 2>&1
for i in 1 2; do run old; done
