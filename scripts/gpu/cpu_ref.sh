python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
python scripts/run_fit_cfg3.py cfg2 500 > gpurun_out/fit_cfg2_refresh.log 2>&1
N=$(grep -o "[0-9]* refreshes" gpurun_out/fit_cfg2_refresh.log | tail -1 | cut -d' ' -f1)
CFG2_REFRESHES=${N:-93} timeout 1800 python scripts/cpu_reference_host.py > gpurun_out/cpu_ref.log 2>&1
