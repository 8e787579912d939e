# pass-1 bound tightening: exactness tests and K-NN timings at two register caps
for mb in 7 6; do rm -f paper_2512_11624_b200/_lib/obj/knn.o; make -s -C paper_2512_11624_b200/csrc EXTRA=-DGSVR_SEL_MINB=$mb >/dev/null 2>&1
 echo "minb=$mb $(grep -A3 k_knn_select paper_2512_11624_b200/_lib/obj/knn.ptxas.log | grep -o 'Used [0-9]* registers\|[0-9]* bytes spill stores' | tr '\n' ' ')"
 for c in cfg2 cfg3; do GSVR_TRACE=1 python scripts/knn_stats.py $c 2>&1 | grep "refresh/knn\|fallback rows" | tail -4 | tr '\n' ' '; echo; done
done > gpurun_out/tighten.log 2>&1
rm -f paper_2512_11624_b200/_lib/obj/knn.o; make -s -C paper_2512_11624_b200/csrc >/dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py -q -p no:cacheprovider -k "refresh or knn or binning" > gpurun_out/tighten_tests.log 2>&1
