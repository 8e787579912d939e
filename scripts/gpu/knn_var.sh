python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
for v in "8 8" "8 6" "12 6"; do set -- $v; rm -f paper_2512_11624_b200/_lib/obj/knn.o
 make -s -C paper_2512_11624_b200/csrc EXTRA="-DGSVR_SEL_CAP=$1 -DGSVR_SEL_MINB=$2" >/dev/null 2>&1
 echo "cap=$1 minb=$2"; GSVR_TRACE=1 python scripts/knn_stats.py cfg3 2>&1 | grep "knn/select\|refresh/knn" | tail -4
done > gpurun_out/knn_var.log
rm -f paper_2512_11624_b200/_lib/obj/knn.o; make -s -C paper_2512_11624_b200/csrc >/dev/null 2>&1
python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py -q -s -k "sampled or seeded or refresh or cfg2_fullsize" 2>&1 | grep -v "^$" | tail -14 > gpurun_out/fullsize.log
