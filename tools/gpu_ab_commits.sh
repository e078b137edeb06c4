# A/B the K1 variants of several commits (repo snapshots under ab/<commit>)
for rep in 1 2; do
for d in ab/d07303b ab/738a503 ab/e982f3a ab/79470be ab/2f088d3 .; do
  for c in llama8k_causal bert512; do
    (cd $d && timeout 120 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > /tmp/x.log 2>&1)
    python -c "
import json
try:
    d=json.loads(open('/tmp/x.log').read().strip().splitlines()[-1]); print('$d', '$c', round(d['config']['kernel_ms']*1e3,1), 'us', round(d['value'],1), d['clocks']['sm_mhz'])
except Exception as e: print('$d $c ERR', open('/tmp/x.log').read()[-300:])
"
  done
done
done
