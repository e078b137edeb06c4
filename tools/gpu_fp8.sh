mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_attention_gpu.py -m gpu -q --timeout 90 -k "e4m3" > gpurun_out/pytest_fp8.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_fp8.log; grep -E "^E  |Error|assert" gpurun_out/pytest_fp8.log | head -12
timeout 120 python bench.py --config llama8k_causal_e4m3 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_fp8.log 2>&1; echo bench=$?
tail -c 1500 gpurun_out/bench_fp8.log
