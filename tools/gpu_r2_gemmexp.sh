# GEMM experiment builds against the product: projection timings (bf16, FP8) and GEMM/FP8 parity
mkdir -p gpurun_out
for L in "" $(cat tools/exp/LIST); do
  echo "== ${L:-product}"
  UH_LIB=${L:+libuhstu_$L.so} timeout 600 python tools/gemm_time.py 2>&1 | grep -v "^pair=0 f1 SiLU B K-major"
  UH_LIB=${L:+libuhstu_$L.so} timeout 600 python tools/fp8_time.py 2>&1 | grep "f1\|f2\|layer"
done
for L in $(cat tools/exp/LIST); do
  UH_TEST_LIB=libuhstu_$L.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fp8.py -x -q -k "gemm or fp8 or layer" 2>&1 | tail -1
done
