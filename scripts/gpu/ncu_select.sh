python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:"k_knn_select" -s 4 -c 1 \
    -o gpurun_out/ncu_select python scripts/knn_stats.py cfg2 > gpurun_out/ncu_select.log 2>&1
