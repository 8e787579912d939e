make -s -C paper_2512_11624_b200/csrc >/dev/null 2>&1
for pc in 3 1.5 6; do echo "per_cell=$pc"; GSVR_KNN_PER_CELL=$pc python scripts/knn_stats.py cfg2 2>&1 | grep -v Warn; done > gpurun_out/knn_time.log
GSVR_TRACE=1 python scripts/knn_stats.py cfg3 >> gpurun_out/knn_time.log 2>&1
rm -rf paper_2512_11624_b200/_lib/obj/knn.o
make -s -C paper_2512_11624_b200/csrc EXTRA=-DGSVR_KNN_STATS >/dev/null 2>&1
for pc in 3 1.5 6; do echo "per_cell=$pc"; GSVR_KNN_PER_CELL=$pc python scripts/knn_stats.py cfg2 2>&1 | grep -v Warn; done > gpurun_out/knn_stats.log
