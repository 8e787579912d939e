python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
python scripts/refresh_only.py cfg2 && \
ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:"k_knn_query|k_bin_hash" -c 2 \
    -o gpurun_out/ncu_refresh_r02 python scripts/refresh_only.py cfg2 > gpurun_out/ncu_refresh.log 2>&1
