python scripts/time_export.py > gpurun_out/export.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "export or rasterize or evaluate" > gpurun_out/export_tests.log 2>&1
