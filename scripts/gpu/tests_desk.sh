set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
python -m pytest tests/test_gpu_render.py tests/test_gpu_fit.py -q -s -k "render or desk" 2>&1 | grep -v "^$" | tail -60 > gpurun_out/desk.log
python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/gputests.log
