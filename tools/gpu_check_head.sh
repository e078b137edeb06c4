# HEAD gate: gpu tests + smoke + attention benches
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -q --timeout 120 -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -5 gpurun_out/pytest_gpu.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()"; echo smoke=$?
for c in llama8k_causal bert512 llama2k_causal llama16k_causal decode32k gemm_chain_e4096; do
  timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.log 2>&1; echo bench_$c=$?
  python -c "
import json
d=json.loads(open('gpurun_out/bench_$c.log').read().strip().splitlines()[-1]); print('$c', d['value'], d['unit'], d.get('roofline',{}).get('frac'), d['config'].get('kernel_ms'))
" 2>&1 | tail -1
done
