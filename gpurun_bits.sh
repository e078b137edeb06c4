mkdir -p gpurun_out/bits
timeout 900 python -m pytest tests/test_attention_gpu.py -k "bit_mask or tensor_mask or causal_mask" -q --timeout 300 > gpurun_out/bits/pytest.log 2>&1; echo bits=$?; tail -3 gpurun_out/bits/pytest.log
timeout 900 python -m pytest tests/test_full_size.py -m gpu -s -q --timeout 600 2>&1 | grep -E "max-abs|passed|failed" > gpurun_out/bits/full_size.txt; cat gpurun_out/bits/full_size.txt
for c in llama4k_mask_bits llama4k_mask_f32; do
 timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bits/b_$c.log 2>&1; echo $c=$?; tail -1 gpurun_out/bits/b_$c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), 'kernel us', round(d['kernel_ms']*1e3,1), 'e2e', round(d['e2e']['value'],1))"
done
