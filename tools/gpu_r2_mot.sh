# NEXT-4 on one B200: MoT parity tests, then the MoT bench line (profiles/r02_mot_bench.json)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_mot.py -x -q 2>&1 | tail -15
timeout 600 python bench.py --config mot --steps 10 --warmup 3 > gpurun_out/r02_mot_bench.json 2> gpurun_out/r02_mot_bench.err
echo "bench rc=$?"; cat gpurun_out/r02_mot_bench.json; tail -5 gpurun_out/r02_mot_bench.err
