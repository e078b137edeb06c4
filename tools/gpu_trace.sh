mkdir -p gpurun_out
NT_LIB_PATH=$PWD/paper_2604_14825_b200/_native/libnt_trace.so python tools/trace_attn.py --cta 0 --out gpurun_out/trace_cta0.json
NT_LIB_PATH=$PWD/paper_2604_14825_b200/_native/libnt_trace.so python tools/trace_attn.py --cta 0 --causal 0 --out gpurun_out/trace_nc_cta0.json
