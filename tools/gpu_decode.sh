mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_decode_gpu.py -m gpu -q --timeout 120 > gpurun_out/pytest_decode.log 2>&1; echo pytest=$?
tail -15 gpurun_out/pytest_decode.log
for c in decode32k decode32k_paged16 decode32k_paged16_hnd decode32k_paged64; do
  timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.log 2>&1; echo bench_$c=$?
  python -c "
import json
d=json.loads(open('gpurun_out/bench_$c.log').read().strip().splitlines()[-1]); r=d['roofline']; print('$c', round(d['config']['kernel_ms']*1e3,1), 'us', round(r['achieved'],1), r['unit'], round(r['frac'],3))
" 2>&1 | tail -1
done
