python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
python -m pytest tests/test_gpu_parity.py tests/test_gpu_fit.py -x -q 2>&1 | tail -2 > gpurun_out/bin_tests.log
for c in cfg2 cfg3; do GSVR_TRACE=1 python scripts/knn_stats.py $c 2>&1 | grep "refresh/bin\|bin/sort\|refresh seeded" | tail -6; done > gpurun_out/bin_time.log
