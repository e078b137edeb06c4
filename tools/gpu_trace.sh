export NT_LIB_PATH=$PWD/paper_2604_14825_b200/_native/libnt_trace.so
python tools/trace_attn.py --cta 0 --item 0 --causal 0 --n 256 --d 64 --b 1 --hq 1 --hkv 1 --scale 1.0 --out gpurun_out/trace_a256.json
python tools/cta_times.py --n 256 --causal 0 --d 64 --hq 1 --hkv 1
