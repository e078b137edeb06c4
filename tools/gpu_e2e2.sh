timeout 300 python -m pytest tests/test_attention_gpu.py -m gpu -q --timeout 90 -x -k "streamed" 2>&1 | tail -2
for c in bert512 llama8k_causal llama2k_causal; do
timeout 120 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$c', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), round(d['e2e']['ms_per_step'],3), 'ms')"
done
