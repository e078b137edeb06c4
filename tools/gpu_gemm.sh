timeout 60 python tools/gemm_ab.py 2>&1 | tail -5
NT_GEMM_1SM=1 timeout 60 python tools/gemm_ab.py 2>&1 | tail -5
timeout 300 python -m pytest tests/test_gemm_gpu.py -m gpu -q --timeout 60 2>&1 | tail -3
