python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -k "refresh or knn or seeded" 2>&1 | tail -2 > gpurun_out/knn_tests.log
for c in cfg2 cfg3; do GSVR_TRACE=1 python scripts/knn_stats.py $c 2>&1 | grep "knn/select\|refresh/knn\|refresh seeded" | tail -6; done > gpurun_out/knn_time.log
