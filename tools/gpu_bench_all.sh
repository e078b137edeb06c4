# Every bench config once (the bench half of tools/gpu_round.sh), into gpurun_out/round/.
mkdir -p gpurun_out/round
cd $GRAFT_REPO_ROOT 2>/dev/null || true
for c in $(python -c "import bench; print(' '.join(bench.CONFIGS))"); do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/round/bench_$c.json.log 2>&1; echo bench_$c=$?
done
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/round/bench_reference.json.log 2>&1; echo ref=$?
