timeout 300 python -m pytest tests/test_attention_gpu.py -q --timeout 120 -x 2>&1 | tail -2
for v in libnautilus_b200.so libnt_poly4.so libnt_poly2.so; do
  for c in llama8k_causal bert512; do
    NT_LIB_PATH=$PWD/paper_2604_14825_b200/_native/$v timeout 120 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > /tmp/x.log 2>&1
    python -c "
import json,sys
try:
    d=json.loads(open('/tmp/x.log').read().strip().splitlines()[-1]); print('$v', '$c', round(d['config']['kernel_ms']*1e3,1), 'us', round(d['value'],1))
except Exception as e: print('$v $c ERR', open('/tmp/x.log').read()[-300:])
"
  done
done
NT_LIB_PATH=$PWD/paper_2604_14825_b200/_native/libnt_trace.so python tools/trace_attn.py --cta 0 --out gpurun_out/trace3_cta0.json > /dev/null 2>&1
