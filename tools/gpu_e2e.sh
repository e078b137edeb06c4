mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_attention_gpu.py -m gpu -q --timeout 300 -k streamed > gpurun_out/pytest_stream.log 2>&1; echo pytest=$?
tail -15 gpurun_out/pytest_stream.log
python tools/e2e_probe.py
