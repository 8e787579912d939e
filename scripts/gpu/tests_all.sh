python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
python -m pytest tests/test_gpu_l1.py -q -s 2>&1 | grep -v "^$" | tail -20 > gpurun_out/l1.log
python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/gputests.log
