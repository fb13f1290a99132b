# backward kernel iteration: parity (attention + layer), timing, experiments
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "bwd or layer or position" > gpurun_out/r2b_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r2b_tests.log
bash tools/gpu_r2_exp.sh
