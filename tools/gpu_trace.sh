mkdir -p gpurun_out
NT_LIB_PATH=$PWD/paper_2604_14825_b200/_native/libnt_trace.so python tools/trace_attn.py --cta ${CTA:-0} --causal 0 --n 512 --d 64 --b 32 --hq 12 --hkv 12 --scale 0.125 --out gpurun_out/trace_bert.json
