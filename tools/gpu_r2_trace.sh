mkdir -p gpurun_out
timeout 300 python tools/trace_fused.py 300 40 1 > gpurun_out/r2t_bwd_rab1.txt 2>&1; echo "bwd rab rc=$?"; tail -8 gpurun_out/r2t_bwd_rab1.txt
timeout 300 python tools/trace_fwd2.py 1 > gpurun_out/r2t_fwd_rab1.txt 2>&1; echo "fwd rab rc=$?"; tail -8 gpurun_out/r2t_fwd_rab1.txt
timeout 1200 python bench.py --config cfg5 --seq-len 4096 --tokens 0 --steps 3 --warmup 3 > gpurun_out/r2_cfg5_L4096.json 2> gpurun_out/r2_cfg5_L4096.err; echo "cfg5 L=4096 rc=$?"; head -c 600 gpurun_out/r2_cfg5_L4096.json; tail -2 gpurun_out/r2_cfg5_L4096.err
timeout 600 python -m pytest tests/test_gpu_stack.py -q 2>&1 | tail -2
