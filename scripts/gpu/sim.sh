python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
python -m pytest tests/test_gpu_simulate.py -q 2>&1 | tail -5 > gpurun_out/sim_tests.log
timeout 600 python scripts/refsim_fit.py 128 0.8 0.8 3.5 200000 0.02 > gpurun_out/refsim.log 2>&1
timeout 600 python scripts/refsim_fit.py 128 0.8 0.8 3.5 70000 0.02 >> gpurun_out/refsim.log 2>&1
timeout 600 python scripts/refsim_fit.py 128 0.8 0.8 3.5 200000 0.0 >> gpurun_out/refsim.log 2>&1
