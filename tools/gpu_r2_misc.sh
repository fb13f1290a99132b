mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/r2m_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r2m_tests.log
bash tools/gpu_r2_exp.sh
