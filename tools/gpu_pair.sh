# CTA-pair GEMM A/B (per shape), GPU tests, bench + launch list; outputs under gpurun_out/
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
for p in 1 0; do UH_GEMM_PAIR=$p timeout 300 python tools/gemm_time.py; done 2>&1 | tee gpurun_out/gemm_pair.log
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench rc=$?"; tail -5 gpurun_out/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
echo "ncu rc=$?"
