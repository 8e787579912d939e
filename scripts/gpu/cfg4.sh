python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
timeout 900 python bench.py --config cfg4 --steps 10 --warmup 3 --no-fit --no-extras --no-cpu-baseline --no-e2e > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err
timeout 900 python scripts/run_fit_cfg3.py cfg4 500 > gpurun_out/fit_cfg4.log 2>&1
timeout 900 python scripts/run_fit_cfg3.py cfg3 500 > gpurun_out/fit_cfg3.log 2>&1
