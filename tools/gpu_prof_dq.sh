# ncu source-level profile of one backward kernel at cfg3 scale (B, RAB, KERN env)
set -x
mkdir -p gpurun_out
timeout 300 python tools/prof_attn.py ${B:-16} ${RAB:-1} > gpurun_out/prof_plain.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on \
    -k regex:"${KERN:-dq}" -s 1 -c 1 -o gpurun_out/prof_${KERN:-dq} \
    python tools/prof_attn.py ${B:-16} ${RAB:-1} > gpurun_out/ncu_k.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/ncu_k.log
