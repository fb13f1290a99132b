# re-entry verification on one B200: GPU tests, smoke, default bench, reference arm
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu > gpurun_out/verify_tests.log 2>&1; tail -3 gpurun_out/verify_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 600 python bench.py > gpurun_out/verify_bench.json 2> gpurun_out/verify_bench.err; tail -c 1500 gpurun_out/verify_bench.json
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/verify_ref.json 2> gpurun_out/verify_ref.err; tail -c 800 gpurun_out/verify_ref.json
