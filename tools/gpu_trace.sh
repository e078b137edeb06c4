mkdir -p gpurun_out
export NT_LIB_PATH=$PWD/paper_2604_14825_b200/_native/libnt_trace.so
python tools/trace_attn.py --cta ${CTA:-0} --item 2 --causal 0 --n 512 --d 64 --b 32 --hq 12 --hkv 12 --scale 0.125 --out gpurun_out/trace_bert_i2.json
python tools/trace_attn.py --cta ${CTA:-0} --item 1 --causal 1 --n 2048 --out gpurun_out/trace_2k_i1.json
