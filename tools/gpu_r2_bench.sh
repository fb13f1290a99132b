# bench line (N=1) + the full GPU test suite + experiment timings
mkdir -p gpurun_out
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err; echo "bench rc=$?"; cat gpurun_out/r2_bench.json | head -c 3000; echo
bash tools/gpu_r2_exp.sh
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/r2_gputests.log 2>&1; echo "gpu tests rc=$?"; tail -4 gpurun_out/r2_gputests.log
