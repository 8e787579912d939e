python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
timeout 1500 python bench.py > gpurun_out/bench_r02c.json 2> gpurun_out/bench_r02c.err
python -m pytest tests -m gpu -q -s > gpurun_out/gputests_full.log 2>&1
tail -4 gpurun_out/gputests_full.log > gpurun_out/gputests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
