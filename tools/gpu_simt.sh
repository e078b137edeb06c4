mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_simt.py -m gpu -q --timeout 300 -x > gpurun_out/pytest_simt.log 2>&1; echo simt=$?
tail -30 gpurun_out/pytest_simt.log
