timeout 1200 python -m pytest tests/test_gpu_init.py -q -s -p no:cacheprovider > gpurun_out/init_tests.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_fit.py tests/test_gpu_multirank.py -q -s -p no:cacheprovider > gpurun_out/init_fit.log 2>&1
