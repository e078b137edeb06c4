# K1 gate + A/B vs the previous commit's library (libprev.so)
mkdir -p gpurun_out
timeout 400 python -m pytest tests/test_attention_gpu.py -m gpu -q --timeout 90 -x > gpurun_out/pytest_k1.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_k1.log
grep -E "^E " gpurun_out/pytest_k1.log | head -8
LIBS="${LIBS:-libprev.so}" CONFIGS="${CONFIGS:-llama8k_causal bert512 llama2k_causal llama16k_causal}" bash tools/gpu_ab_libs.sh
[ -n "$TRACE" ] && bash tools/gpu_trace.sh > gpurun_out/trace.log 2>&1
true
