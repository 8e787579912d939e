rm -f paper_2512_11624_b200/_lib/obj/batch.o; make -s -C paper_2512_11624_b200/csrc EXTRA=-DGSVR_BIN_PROFILE >/dev/null 2>&1
for c in cfg2 cfg3; do python scripts/knn_stats.py $c 2>&1 | grep "BINPHASE" | tail -3; done > gpurun_out/binprof.log 2>&1
rm -f paper_2512_11624_b200/_lib/obj/batch.o; make -s -C paper_2512_11624_b200/csrc >/dev/null 2>&1
