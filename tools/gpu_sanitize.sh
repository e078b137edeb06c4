# compute-sanitizer over every kernel family at small shapes.
mkdir -p gpurun_out/sanitize
cd $GRAFT_REPO_ROOT 2>/dev/null || true
timeout 300 python tools/sanitize_cases.py > gpurun_out/sanitize/plain.log 2>&1; echo plain=$?
for tool in memcheck synccheck initcheck racecheck; do
  for fam in k1 k2 k3 chain simt; do
    timeout 900 compute-sanitizer --tool $tool --print-limit 20 --error-exitcode 9 \
      python tools/sanitize_cases.py $fam > gpurun_out/sanitize/${tool}_${fam}.log 2>&1
    echo ${tool}_${fam}=$?
    tail -2 gpurun_out/sanitize/${tool}_${fam}.log
  done
done
