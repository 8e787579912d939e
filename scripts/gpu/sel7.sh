for mb in 6 7 8; do rm -f paper_2512_11624_b200/_lib/obj/knn.o; make -s -C paper_2512_11624_b200/csrc EXTRA=-DGSVR_SEL_MINB=$mb >/dev/null 2>&1
 echo "minb=$mb $(grep -A3 k_knn_select paper_2512_11624_b200/_lib/obj/knn.ptxas.log | grep -o 'Used [0-9]* registers\|[0-9]* bytes spill stores' | tr '\n' ' ')"
 for c in cfg2 cfg3; do GSVR_TRACE=1 python scripts/knn_stats.py $c 2>&1 | grep "refresh/knn" | tail -2 | tr '\n' ' '; echo; done
done > gpurun_out/sel7.log 2>&1
rm -f paper_2512_11624_b200/_lib/obj/knn.o; make -s -C paper_2512_11624_b200/csrc >/dev/null 2>&1
