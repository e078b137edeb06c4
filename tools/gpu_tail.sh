timeout 600 python -m pytest tests/test_attention_gpu.py -m gpu -q --timeout 120 -x > gpurun_out/pytest_tail.log 2>&1; echo pytest=$?
tail -2 gpurun_out/pytest_tail.log; grep -E "^E  " gpurun_out/pytest_tail.log | head -8
for rep in 1 2; do for v in on off; do
  if [ $v = off ]; then export NT_ATTN_NO_TAIL_SPLIT=1; else unset NT_ATTN_NO_TAIL_SPLIT; fi
  timeout 120 python bench.py --config bert512 --steps 20 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('tail-$v bert512', round(d['config']['kernel_ms']*1e3,1), round(d['value'],1), d['gpu_launches'])"
done; done
