python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
for u in 4 8 2; do rm -f paper_2512_11624_b200/_lib/obj/knn.o; make -s -C paper_2512_11624_b200/csrc EXTRA=-DGSVR_KNN_UNROLL=$u >/dev/null 2>&1
 echo "unroll=$u $(grep -A3 k_knn_select paper_2512_11624_b200/_lib/obj/knn.ptxas.log | grep -o 'Used [0-9]* registers\|[0-9]* bytes spill stores' | tr '\n' ' ')"
 for c in cfg2 cfg3; do GSVR_TRACE=1 python scripts/knn_stats.py $c 2>&1 | grep "refresh/knn" | tail -2 | tr '\n' ' '; echo; done
done
rm -f paper_2512_11624_b200/_lib/obj/knn.o; make -s -C paper_2512_11624_b200/csrc >/dev/null 2>&1
