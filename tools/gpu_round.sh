# Round gate on one B200: GPU tests, smoke, every bench config (with CPU baseline),
# the reference arm, ncu captures of each kernel family and the default launch list.
mkdir -p gpurun_out/round
cd $GRAFT_REPO_ROOT 2>/dev/null || true
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/round/nvidia_smi.txt
timeout 1500 python -m pytest tests -m gpu -q --timeout 300 > gpurun_out/round/pytest_gpu.log 2>&1; echo pytest=$?
tail -3 gpurun_out/round/pytest_gpu.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/round/smoke.log 2>&1; echo smoke=$?
for c in llama8k_causal llama2k_causal llama4k_causal llama16k_causal llama8k_causal_1group llama8k_causal_e4m3 llama4k_mask_bits llama4k_mask_f32 bert512 attn256 decode32k decode32k_paged16 decode32k_paged16_hnd decode32k_paged64 decode32k_e4m3 decode32k_e4m3_paged16 decode32k_e4m3_paged64 decode64k decode128k gemm_chain_e4096 gemm_chain_e128; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/round/bench_$c.json.log 2>&1; echo bench_$c=$?
done
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/round/bench_reference.json.log 2>&1; echo ref=$?
timeout 600 python tools/tune_compare.py --prog scaled_0p125 --bind N=512,M=512,D=64 --outer 32,12,12 > gpurun_out/round/tune_bert512.json 2>/dev/null; echo tune_bert=$?
timeout 900 python tools/tune_compare.py --prog llama_causal --bind N=8192,M=8192,D=128 --outer 1,32,8 --causal --budget 32 > gpurun_out/round/tune_causal8k.json 2>/dev/null; echo tune_8k=$?
python tools/latency_probe.py > gpurun_out/round/latency_attn256.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/round/launches_llama8k.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo launches=$?
# cap NAME KERNEL_REGEX SKIP CONFIG [summary args]: one --set full capture, summarised on
# the box (tools/ncu_summary.py); only the headline report is kept (gpurun_out <= 64 MiB)
cap() {
  name=$1; k=$2; skip=$3; cfg=$4; shift 4
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s $skip -c 1 -o gpurun_out/round/$name python bench.py --config $cfg --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/round/ncu_$name.log 2>&1; echo ncu_$name=$?
  python tools/ncu_summary.py gpurun_out/round/$name.ncu-rep gpurun_out/round/${name}_ncu.json --workload $cfg "$@" > /dev/null 2>&1
  ncu -i gpurun_out/round/$name.ncu-rep --page source --csv --print-source sass > gpurun_out/round/${name}_sass.csv 2>/dev/null
  python tools/ncu_sass_stalls.py gpurun_out/round/${name}_sass.csv --top 30 > gpurun_out/round/${name}_stalls.txt 2>&1
  rm -f gpurun_out/round/${name}_sass.csv
  [ "$name" = attn_llama8k ] || rm -f gpurun_out/round/$name.ncu-rep
}
cap attn_llama8k attn_fwd 3 llama8k_causal --algorithmic-bytes 167772160 --algorithmic-flops 549822922752
cap attn_bert512 attn_fwd 3 bert512 --algorithmic-bytes 100663296 --algorithmic-flops 25769803776
cap decode32k decode_tc 3 decode32k --algorithmic-bytes 8590983168
cap decode32k_paged16 decode_tc 3 decode32k_paged16 --algorithmic-bytes 8590983168
cap decode32k_e4m3 decode_tc 3 decode32k_e4m3 --algorithmic-bytes 4295753728
cap gemm4k gemm2_kernel 6 gemm_chain_e4096 --algorithmic-flops 137438953472
cap attn_llama8k_e4m3 attn_fwd 3 llama8k_causal_e4m3 --algorithmic-bytes 117440512 --algorithmic-flops 549822922752
cap gemm_e128 gemm_kernel 3 gemm_chain_e128 --algorithmic-flops 4294967296
cap attn_1group attn_fwd 3 llama8k_causal_1group --algorithmic-flops 68727865344
ls -la gpurun_out/round | head -40
