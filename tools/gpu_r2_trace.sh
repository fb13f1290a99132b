mkdir -p gpurun_out
timeout 300 python tools/trace_fused.py 300 40 1 > gpurun_out/r2t_bwd_rab1.txt 2>&1; echo "bwd rab rc=$?"
timeout 300 python tools/trace_fused.py 300 40 0 > gpurun_out/r2t_bwd_rab0.txt 2>&1; echo "bwd norab rc=$?"
tail -8 gpurun_out/r2t_bwd_rab1.txt; tail -8 gpurun_out/r2t_bwd_rab0.txt
