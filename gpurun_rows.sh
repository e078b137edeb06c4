for c in llama2k_causal attn256 llama8k_causal_1group bert512 llama16k_causal; do
 for r in 256 128; do
  timeout 300 python bench.py --config $c --item-rows $r --steps 10 --warmup 3 --no-cpu-baseline > /tmp/b.log 2>&1
  python - "$c" "$r" <<'PY'
import json,sys
try:
    d=json.loads(open("/tmp/b.log").read().strip().splitlines()[-1])
    print(sys.argv[1], sys.argv[2], round(d["value"],1), "kernel_us", round(d["kernel_ms"]*1e3,1), "ctas/sm", d.get("k1_ctas_per_sm"))
except Exception as e: print(sys.argv[1], sys.argv[2], "ERR", e, open("/tmp/b.log").read()[-500:])
PY
 done
done
