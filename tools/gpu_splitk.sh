timeout 300 python -m pytest tests/test_gemm_gpu.py -m gpu -q --timeout 60 -x 2>&1 | tail -3
for c in gemm_chain_e128 gemm_chain_e4096; do
timeout 120 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$c', round(d['config']['kernel_ms']*1e3,1), round(d['value'],1), round(d['roofline']['frac'],3), d['gpu_launches'])"
done
