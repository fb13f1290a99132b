# full GPU test suite + attention timing
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/r2_gputests.log 2>&1; echo "gpu tests rc=$?"; tail -25 gpurun_out/r2_gputests.log
timeout 600 python tools/attn_time.py > gpurun_out/r2_time.log 2>&1; grep "B=" gpurun_out/r2_time.log
