mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 300 python tools/fp8_time.py 2>&1 | tee gpurun_out/fp8_time2.log
UH_GEMM_PAIR=0 timeout 300 python tools/gemm_time.py 2>&1 | tee gpurun_out/gemm_time2.log
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 | tee gpurun_out/gpu_tests.log
timeout 900 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_dbuf.json 2> gpurun_out/bench_dbuf.err
python -c "import json;d=json.load(open('gpurun_out/bench_dbuf.json'));print(d['value'],d['ms_per_step'])"
