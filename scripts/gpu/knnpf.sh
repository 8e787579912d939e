for c in cfg2 cfg3; do GSVR_TRACE=1 python scripts/knn_stats.py $c 2>&1 | grep "refresh/knn" | tail -2 | tr '\n' ' '; echo; done > gpurun_out/knnpf.log 2>&1
timeout 900 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py -q -p no:cacheprovider -k "refresh or knn" > gpurun_out/knnpf_tests.log 2>&1
