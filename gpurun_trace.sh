mkdir -p gpurun_out/trace
export NT_LIB_PATH=$PWD/paper_2604_14825_b200/_native/libnt_trace.so
for it in 0 1 2 3 4; do
python tools/trace_attn.py --b 32 --hq 12 --hkv 12 --n 512 --d 64 --causal 0 --scale 0.125 --item $it --out gpurun_out/trace/bert_item$it.json
done
python tools/cta_times.py --b 32 --hq 12 --hkv 12 --n 512 --d 64 --causal 0
python tools/trace_attn.py --item 3 --out gpurun_out/trace/l8k_item3.json
python tools/cta_times.py --n 8192
