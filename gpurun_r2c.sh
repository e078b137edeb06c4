mkdir -p gpurun_out/r2c
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 > gpurun_out/r2c/pytest_gpu.log 2>&1; echo pytest=$?; tail -4 gpurun_out/r2c/pytest_gpu.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2c/smoke.log 2>&1; echo smoke=$?; tail -1 gpurun_out/r2c/smoke.log
timeout 600 python tools/tune_compare.py --prog scaled_0p125 --bind N=512,M=512,D=64 --outer 32,12,12 > gpurun_out/r2c/tune_bert512.json 2> gpurun_out/r2c/tune_bert512.err; echo tune_bert=$?; tail -c 1500 gpurun_out/r2c/tune_bert512.json
timeout 900 python tools/tune_compare.py --prog llama_causal --bind N=2048,M=2048,D=128 --outer 1,32,8 --causal > gpurun_out/r2c/tune_causal2k.json 2> gpurun_out/r2c/tune_causal2k.err; echo tune_2k=$?; tail -c 1500 gpurun_out/r2c/tune_causal2k.json
timeout 900 compute-sanitizer --tool initcheck --print-limit 20 --error-exitcode 9 python tools/sanitize_cases.py k1 > gpurun_out/r2c/initcheck_k1.log 2>&1; echo initcheck_k1=$?; tail -2 gpurun_out/r2c/initcheck_k1.log
