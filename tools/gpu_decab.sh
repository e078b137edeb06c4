timeout 300 python -m pytest tests/test_decode_gpu.py -m gpu -q --timeout 60 -x 2>&1 | tail -2
for rep in 1 2; do for v in libnautilus_b200.so $LIBS; do for c in decode32k decode32k_paged16 decode32k_paged16_hnd decode32k_paged64; do
NT_LIB_PATH=$PWD/paper_2604_14825_b200/_native/$v timeout 120 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v', '$c', round(d['config']['kernel_ms']*1e3,1), round(d['roofline']['frac'],3))"
done; done; done
