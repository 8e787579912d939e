python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
python scripts/refresh_only.py cfg2 >/dev/null 2>&1 && \
ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:"k_knn_select" -c 1 \
    -o gpurun_out/ncu_select_r02 python scripts/refresh_only.py cfg2 > gpurun_out/ncu_sel.log 2>&1
ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:"k_bin_hash" -c 1 \
    -o gpurun_out/ncu_binhash_r02 python scripts/refresh_only.py cfg2 > gpurun_out/ncu_bin.log 2>&1
