# launch list of the bench step + ncu --set full of the fused attention backward (cfg3, rab on)
mkdir -p gpurun_out
bash tools/gpu_bench.sh > /dev/null 2>&1
timeout 300 python tools/prof_attn.py 16 1 > gpurun_out/prof_plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"fused|dq_finish" -c 2 \
    -o gpurun_out/prof_fused python tools/prof_attn.py 16 1 > gpurun_out/ncu_fused.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/ncu_fused.log
