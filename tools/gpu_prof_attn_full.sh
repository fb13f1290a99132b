# ncu --set full of the three attention kernels at cfg3 (B=16, rab on): fwd, dq, dkv
set -x
mkdir -p gpurun_out
timeout 300 python tools/prof_attn.py 16 1 > gpurun_out/prof_plain.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"attn_" -s 3 -c 3 \
    -o gpurun_out/prof_attn16 python tools/prof_attn.py 16 1 > gpurun_out/ncu_attn16.log 2>&1
echo "ncu rc=$?"
