for i in 1 2; do timeout 60 python tools/k1_stress.py 1 32 8192 128 1 0 100 2>&1 | grep -v Warning | tail -1; done
timeout 60 python tools/k1_stress.py 32 12 512 128 0 0 400 2>&1 | grep -v Warning | tail -1
timeout 60 python tools/k1_stress.py 4 32 2048 128 1 1 400 2>&1 | grep -v Warning | tail -1
TRACE=1 bash tools/gpu_k1.sh
