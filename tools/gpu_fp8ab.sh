for rep in 1 2; do for v in libnautilus_b200.so $LIBS; do
NT_LIB_PATH=$PWD/paper_2604_14825_b200/_native/$v timeout 120 python bench.py --config llama8k_causal_e4m3 --steps 20 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['config']['kernel_ms']*1e3,1), round(d['value'],1))"
done; done
