python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
B="python bench.py --steps 2 --warmup 3 --no-fit --no-cpu-baseline --no-extras --no-e2e"
$B > gpurun_out/b_plain.json 2>/dev/null
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r02.csv $B > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:"k_train_planar" --launch-skip 3 -c 1 \
    -o gpurun_out/ncu_tp_r02 $B > gpurun_out/ncu_tp.log 2>&1
ncu --set full --clock-control none -k regex:"k_gather_grads|k_field_step|k_slice_step|k_pack_grec|k_disp_bounds|k_disp_points|k_slice_reduce" \
    --launch-skip 14 -c 7 -o gpurun_out/ncu_epoch_r02 $B > gpurun_out/ncu_epoch.log 2>&1
python scripts/refresh_only.py cfg2 >/dev/null 2>&1 && \
ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:"k_knn_select" -c 1 \
    -o gpurun_out/ncu_select_r02 python scripts/refresh_only.py cfg2 > gpurun_out/ncu_sel.log 2>&1
ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:"k_bin_hash" -c 1 \
    -o gpurun_out/ncu_binhash_r02 python scripts/refresh_only.py cfg2 > gpurun_out/ncu_bin.log 2>&1
python scripts/setup_only.py cfg3 >/dev/null 2>&1 && \
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_setup_r02.csv python scripts/setup_only.py cfg3 > gpurun_out/ncu_setup.log 2>&1
