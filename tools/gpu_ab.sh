# A/B of library builds on one box: bash tools/gpu_ab.sh <variant> ... runs bench configs with
# NT_LIB_PATH=ab/lib_<variant>.so (build them with build.build(defines=[...], out="ab/lib_<v>.so")), twice each.
mkdir -p gpurun_out/ab
for rep in 1 2; do
for v in "$@"; do
  for c in bert512 llama8k_causal llama2k_causal llama8k_causal_1group; do
    NT_LIB_PATH=$PWD/ab/lib_$v.so timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ab/${v}_${c}_$rep.log 2>&1
    python - "$v" "$c" "$rep" <<'PY'
import json,sys
v,c,r=sys.argv[1:]
try:
    d=json.loads(open(f"gpurun_out/ab/{v}_{c}_{r}.log").read().strip().splitlines()[-1])
    print(f"{v:8s} {c:22s} rep{r} {d['value']:7.1f} TF  kernel {d['kernel_ms']*1e3:7.1f} us")
except Exception as e: print(v, c, "ERR", e)
PY
  done
done
done
