# K3 A/B: default library vs $LIBS variants (tools/gemm_ab.py), cuBLAS for context
timeout 300 python -m pytest tests/test_gemm_gpu.py -m gpu -q --timeout 60 -x 2>&1 | tail -2
for v in libnautilus_b200.so $LIBS; do
  echo "== $v"; NT_LIB_PATH=$PWD/paper_2604_14825_b200/_native/$v timeout 60 python tools/gemm_ab.py 2>&1 | tail -4
done
timeout 60 python tools/cublas_ref.py 2>&1 | tail -3
