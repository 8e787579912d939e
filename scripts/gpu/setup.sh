python scripts/time_setup.py cfg3 > gpurun_out/setup_cfg3.log 2>&1
python scripts/time_setup.py cfg2 > gpurun_out/setup_cfg2.log 2>&1
timeout 600 python -m pytest tests/test_gpu_init.py -q -s -p no:cacheprovider -k "cumsum or cfg3" > gpurun_out/init_tests.log 2>&1
