# round-2 baseline: attention timings (rab on/off), then the GPU test suite
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/r2_base_smi.txt
timeout 600 python tools/attn_time.py > gpurun_out/r2_base_attn.log 2>&1; echo "attn rc=$?"
cat gpurun_out/r2_base_attn.log
timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/r2_base_tests.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/r2_base_tests.log
