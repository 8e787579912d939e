python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 900 python scripts/diag_cfg2_fit.py > gpurun_out/diag_cfg2.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_r02a.json 2> gpurun_out/bench_r02a.err
