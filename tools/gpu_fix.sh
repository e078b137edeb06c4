timeout 600 python -m pytest tests/test_attention_gpu.py -m gpu -q --timeout 120 -x > gpurun_out/pytest_fix.log 2>&1; echo pytest=$?
tail -2 gpurun_out/pytest_fix.log; grep -E "^E  " gpurun_out/pytest_fix.log | head -8
python tools/split_probe.py 2>&1 | sed -n '1p;5p'
for a in "1 4 8192 128 1 0 60" "1 2 4096 128 0 1 100" "2 1 3000 64 1 0 100"; do timeout 120 python tools/k1_stress.py $a 2>&1 | tail -1; done
