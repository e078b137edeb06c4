# Round gate on one B200: GPU tests, smoke, every bench config (with CPU baseline),
# the reference arm, ncu captures of each kernel family and the default launch list.
mkdir -p gpurun_out/round
cd $GRAFT_REPO_ROOT 2>/dev/null || true
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/round/nvidia_smi.txt
timeout 1500 python -m pytest tests -m gpu -q --timeout 300 > gpurun_out/round/pytest_gpu.log 2>&1; echo pytest=$?
tail -3 gpurun_out/round/pytest_gpu.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/round/smoke.log 2>&1; echo smoke=$?
for c in llama8k_causal llama2k_causal llama16k_causal llama8k_causal_1group llama8k_causal_e4m3 bert512 attn256 decode32k decode32k_paged16 decode32k_paged16_hnd decode32k_paged64 gemm_chain_e4096 gemm_chain_e128; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/round/bench_$c.json.log 2>&1; echo bench_$c=$?
done
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/round/bench_reference.json.log 2>&1; echo ref=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/round/launches_llama8k.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo launches=$?
cap() { timeout 600 ncu --set full --clock-control none --import-source on -k regex:$2 -s $3 -c 1 -o gpurun_out/round/$1 python bench.py --config $4 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/round/ncu_$1.log 2>&1; echo ncu_$1=$?; }
cap attn_llama8k attn_fwd 3 llama8k_causal
cap attn_bert512 attn_fwd 3 bert512
cap decode32k decode_split 3 decode32k
cap decode32k_paged16 decode_split 3 decode32k_paged16
cap gemm4k gemm2_kernel 6 gemm_chain_e4096
cap attn_llama8k_e4m3 attn_fwd 3 llama8k_causal_e4m3
cap gemm_e128 gemm_kernel 3 gemm_chain_e128
ls -la gpurun_out/round | head -40
