mkdir -p gpurun_out
export NT_LIB_PATH=$PWD/paper_2604_14825_b200/_native/libnt_trace.so
python tools/trace_attn.py --cta ${CTA:-0} --item 1 --causal 1 --n 8192 --out gpurun_out/trace_8k_i1.json
python tools/trace_attn.py --cta ${CTA:-0} --item 1 --causal 1 --n 8192 --e4m3 --out gpurun_out/trace_8k_fp8_i1.json
