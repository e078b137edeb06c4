# A/B library variants (NT_LIB_PATH) on the attention configs
for rep in 1 2; do
for v in libnautilus_b200.so $LIBS; do
  for c in $CONFIGS; do
    NT_LIB_PATH=$PWD/paper_2604_14825_b200/_native/$v timeout 120 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > /tmp/x.log 2>&1
    python -c "
import json
try:
    d=json.loads(open('/tmp/x.log').read().strip().splitlines()[-1]); print('$v', '$c', round(d['config']['kernel_ms']*1e3,1), 'us', round(d['value'],1))
except Exception as e: print('$v $c ERR', open('/tmp/x.log').read()[-300:])
"
  done
done
done
