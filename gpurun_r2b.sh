mkdir -p gpurun_out/r2b
timeout 600 python -m pytest tests/test_attention_gpu.py -k "item_rows" -q --timeout 300 > gpurun_out/r2b/pytest_nq1.log 2>&1; echo nq1=$?; tail -3 gpurun_out/r2b/pytest_nq1.log
for c in bert512 llama8k_causal llama8k_causal_1group; do
 for r in 256 128; do
  timeout 300 python bench.py --config $c --item-rows $r --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2b/b_${c}_$r.log 2>&1
  python - "$c" "$r" <<'PY'
import json,sys
try:
    d=json.loads(open(f"gpurun_out/r2b/b_{sys.argv[1]}_{sys.argv[2]}.log").read().strip().splitlines()[-1])
    print(sys.argv[1], sys.argv[2], round(d["value"],1), "kernel_us", round(d["kernel_ms"]*1e3,1), "frac", round(d["roofline"]["frac"],3), "ctas/sm", d.get("k1_ctas_per_sm"))
except Exception as e: print(sys.argv[1], sys.argv[2], "ERR", e)
PY
 done
done
