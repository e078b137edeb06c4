mkdir -p gpurun_out
export NT_LIB_PATH=$PWD/paper_2604_14825_b200/_native/libnt_trace.so
python tools/trace_attn.py --cta ${CTA:-0} --item 1 --causal 1 --n 8192 --hq 4 --hkv 1 --out gpurun_out/trace_split_i1.json
python tools/cta_times.py --hq 4 --hkv 1 --n 8192 2>&1 | tail -15
