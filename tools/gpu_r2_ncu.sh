# ncu --set full of the attention kernels at cfg3 (rab on, P = 16384)
mkdir -p gpurun_out
timeout 300 python tools/prof_attn.py 16 1 > gpurun_out/r2n_plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"attn_fwd|attn_bwd_fused|dq_finish|rab_ext" -c 4 \
   -o gpurun_out/r2n_attn python tools/prof_attn.py 16 1 > gpurun_out/r2n_ncu.log 2>&1; echo "ncu rc=$?"; tail -3 gpurun_out/r2n_ncu.log
