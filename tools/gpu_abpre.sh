for rep in 1 2; do
for c in bert512 llama8k_causal llama2k_causal; do
  timeout 120 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('new', '$c', round(d['config']['kernel_ms']*1e3,1))"
  (cd tmp_pre && timeout 120 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('pre', '$c', round(d['config']['kernel_ms']*1e3,1))")
done; done
