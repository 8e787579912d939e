python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
python -m pytest tests/test_gpu_parity.py -q -s -k "refresh or knn" 2>&1 | grep -v "^$" | tail -12 > gpurun_out/knn_tests.log
python -m pytest tests/test_gpu_fullsize.py -q -s -k seeded 2>&1 | grep -v "^$" | tail -12 >> gpurun_out/knn_tests.log
for sel in 1 0; do echo "GSVR_KNN_SELECT=$sel"; GSVR_KNN_SELECT=$sel GSVR_TRACE=1 python scripts/knn_stats.py cfg2 2>&1 | grep -v Warn | grep "refresh\|knn" ; done > gpurun_out/knn_time.log
for sel in 1 0; do echo "GSVR_KNN_SELECT=$sel"; GSVR_KNN_SELECT=$sel GSVR_TRACE=1 python scripts/knn_stats.py cfg3 2>&1 | grep -v Warn | grep "refresh\|knn" ; done >> gpurun_out/knn_time.log
