for c in cfg2 cfg3 cfg4; do for gp in 0 1 0 1; do
 r=$(GSVR_GPOS=$gp timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-fit --no-extras --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(round(d['value']/1e9,3), 'G px/s kern', round(d['roofline']['kernel_ms'],3), 'frac', round(d['roofline']['frac'],4))")
 echo "$c gpos=$gp $r"
done; done > gpurun_out/gpos.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_fit.py -q -p no:cacheprovider -x > gpurun_out/gpos_tests.log 2>&1
