python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
python scripts/run_fit_cfg3.py 2>&1 | tail -5 > gpurun_out/fit3.log
GSVR_KNN_SELECT=0 python scripts/run_fit_cfg3.py 2>&1 | tail -5 >> gpurun_out/fit3.log
