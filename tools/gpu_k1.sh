# K1 gate: attention GPU tests + benches (+ optional trace)
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_attention_gpu.py -m gpu -q --timeout 60 -x > gpurun_out/pytest_k1.log 2>&1; echo pytest=$?
tail -5 gpurun_out/pytest_k1.log
grep -E "^E " gpurun_out/pytest_k1.log | head -5
for c in llama8k_causal bert512 llama2k_causal llama16k_causal attn256; do
  timeout 120 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.log 2>&1; echo bench_$c=$?
  python -c "
import json
d=json.loads(open('gpurun_out/bench_$c.log').read().strip().splitlines()[-1]); print('$c', round(d['config']['kernel_ms']*1e3,1), 'us', round(d['value'],1), d['unit'], round(d['roofline']['frac'],3), 'e2e', round(d['e2e']['value'],1), d['clocks'])
" 2>&1 | tail -1
done
if [ -n "$TRACE" ]; then
NT_LIB_PATH=$PWD/paper_2604_14825_b200/_native/libnt_trace.so timeout 60 python tools/trace_attn.py --cta 0 --causal 0 --out gpurun_out/trace_nc.json | tail -30
fi
