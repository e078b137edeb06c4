# K1 stress sweep: each config in its own process under a timeout
while read -r args; do
  timeout 120 python tools/k1_stress.py $args 2>&1 | tail -1
done <<'CFG'
1 32 8192 128 1 0 100
1 32 2048 128 1 0 300
32 12 512 64 0 0 300
32 12 512 64 0 1 200
4 8 1000 64 1 1 200
1 32 8192 128 1 0 100 1
2 16 1536 128 0 1 200 1
1 4 129 128 1 1 300
1 1 64 64 0 0 300
3 5 777 128 0 0 200
CFG
