# round 2: CTA-0 timelines of the fused backward and the forward (trace builds), rab on and off
mkdir -p gpurun_out
timeout 300 python tools/trace_fused.py 300 40 1 > gpurun_out/r2t_bwd_rab1.txt 2>&1; echo "bwd rab rc=$?"
timeout 300 python tools/trace_fused.py 300 40 0 > gpurun_out/r2t_bwd_rab0.txt 2>&1; echo "bwd norab rc=$?"
timeout 300 python tools/trace_fwd2.py 1 > gpurun_out/r2t_fwd_rab1.txt 2>&1; echo "fwd rab rc=$?"
timeout 300 python tools/trace_fwd2.py 0 > gpurun_out/r2t_fwd_rab0.txt 2>&1; echo "fwd norab rc=$?"
tail -12 gpurun_out/r2t_bwd_rab0.txt
