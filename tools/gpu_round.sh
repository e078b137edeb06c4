# full GPU gate + per-kernel ncu captures (one GPU, short commands)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 300 > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_gpu.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()"; echo smoke=$?
for c in llama8k_causal bert512 decode32k gemm_chain_e4096 gemm_chain_e128 attn256 llama2k_causal llama16k_causal; do
  timeout 300 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/bench_$c.log 2>&1; echo bench_$c=$?
done
timeout 300 ncu --set full --clock-control none --import-source on -k regex:decode_split -s 3 -c 1 -o gpurun_out/decode32k python bench.py --config decode32k --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_decode.log 2>&1; echo ncu_decode=$?
timeout 300 ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 6 -c 1 -o gpurun_out/gemm4k python bench.py --config gemm_chain_e4096 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_gemm.log 2>&1; echo ncu_gemm=$?
timeout 300 ncu --set full --clock-control none --import-source on -k regex:attn_fwd -s 3 -c 1 -o gpurun_out/attn8k python bench.py --config llama8k_causal --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_attn.log 2>&1; echo ncu_attn=$?
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches_llama8k.csv python bench.py --config llama8k_causal --steps 5 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo ncu_launches=$?
