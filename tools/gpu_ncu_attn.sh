mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_fwd -s 3 -c 1 -o gpurun_out/attn8k_persist python bench.py --config llama8k_causal --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_attn.log 2>&1; echo ncu_attn=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_fwd -s 3 -c 1 -o gpurun_out/bert_persist python bench.py --config bert512 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_bert.log 2>&1; echo ncu_bert=$?
tail -3 gpurun_out/ncu_attn.log
