mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_attention_gpu.py -m gpu -q --timeout 300 -k streamed > gpurun_out/pytest_stream.log 2>&1; echo pytest=$?
tail -15 gpurun_out/pytest_stream.log
for c in llama8k_causal bert512 decode32k; do
  timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.log 2>&1; echo bench_$c=$?
  python -c "
import json
d=json.loads(open('gpurun_out/bench_$c.log').read().strip().splitlines()[-1]); print('$c', round(d['value'],1), d['unit'], 'e2e', round(d['e2e']['value'],2), round(d['e2e']['ms_per_step'],3), 'ms')
" 2>&1 | tail -1
done
