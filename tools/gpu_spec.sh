# K1 speculative-max gate: attention GPU tests, then A/B against the max-first build
mkdir -p gpurun_out
timeout 400 python -m pytest tests/test_attention_gpu.py -m gpu -q --timeout 90 -x > gpurun_out/pytest_k1.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_k1.log
grep -E "^E " gpurun_out/pytest_k1.log | head -8
LIBS="${LIBS:-libspec0.so}" CONFIGS="${CONFIGS:-llama8k_causal bert512 llama2k_causal llama16k_causal}" bash tools/gpu_ab_libs.sh
