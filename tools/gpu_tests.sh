mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 300 > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
grep -E "passed|failed|error" gpurun_out/pytest_gpu.log | tail -5
grep -E "^(FAILED|ERROR)" gpurun_out/pytest_gpu.log | head -20
