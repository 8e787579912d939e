timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -p no:cacheprovider -k "refresh or binning or bin" > gpurun_out/bin7_tests.log 2>&1
for c in cfg2 cfg3; do echo "$c $(GSVR_TRACE=1 python scripts/knn_stats.py $c 2>&1 | grep 'refresh/bin' | tail -1)"; done > gpurun_out/bin7.log 2>&1
