python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
timeout 900 python bench.py > gpurun_out/bench_r02b.json 2> gpurun_out/bench_r02b.err
python -m pytest tests/test_gpu_bench.py -q -s 2>&1 | tail -30 > gpurun_out/bench_test.log
