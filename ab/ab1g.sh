for rep in 1 2; do for ir in 256 128; do for c in llama8k_causal_1group llama2k_causal; do
timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --item-rows $ir 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c rows $ir', round(d['value'],1), round(d['kernel_ms']*1e3,2))"
done; done; done
