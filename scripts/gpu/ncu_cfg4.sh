python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
ncu --set full --clock-control none -k regex:"k_train_planar" --launch-skip 3 -c 1 -o gpurun_out/ncu_tp_cfg4 \
  python bench.py --config cfg4 --steps 2 --warmup 3 --no-fit --no-extras --no-cpu-baseline --no-e2e > gpurun_out/ncu_cfg4.log 2>&1
