mkdir -p gpurun_out/ncu
for c in bert512 llama8k_causal; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_fwd -s 3 -c 1 -o gpurun_out/ncu/$c python bench.py --config $c --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu/$c.log 2>&1; echo ncu_$c=$?
ncu -i gpurun_out/ncu/$c.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu/${c}_sass.csv 2>&1; echo src=$?
ncu -i gpurun_out/ncu/$c.ncu-rep --page raw --csv > gpurun_out/ncu/${c}_raw.csv 2>&1
done
ls -la gpurun_out/ncu
