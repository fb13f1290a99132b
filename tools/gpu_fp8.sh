# NEXT-2 FP8: GPU parity (fp8 + GEMM pair cases), timing; outputs under gpurun_out/
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_fp8.py -x -q 2>&1 | tail -15 | tee gpurun_out/fp8_tests.log
timeout 300 python tools/fp8_time.py 2>&1 | tee gpurun_out/fp8_time.log
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 | tee gpurun_out/gpu_tests.log
