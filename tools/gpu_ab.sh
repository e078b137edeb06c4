# A/B: attention softmax exp2 variants + decode kernel; correctness first
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q --timeout 120 -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_gpu.log
for v in libnt_poly0.so libnt_poly8.so libnautilus_b200.so libnt_poly2.so; do
  for c in llama8k_causal bert512; do
    NT_LIB_PATH=$PWD/paper_2604_14825_b200/_native/$v timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/ab_${v}_$c.log 2>&1
    python - "$v" "$c" gpurun_out/ab_${v}_$c.log <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[3]).read().strip().splitlines()[-1]); print(sys.argv[1], sys.argv[2], round(d["value"],1), round(d["roofline"]["frac"],3), d["clocks"]["sm_mhz"])
except Exception as e: print(sys.argv[1], sys.argv[2], "ERR", open(sys.argv[3]).read()[-500:])
PY
  done
done
timeout 300 python bench.py --config decode32k --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_decode32k.log 2>&1; tail -1 gpurun_out/bench_decode32k.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('decode', d['roofline'])"
