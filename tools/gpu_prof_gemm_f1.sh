# f1 GEMM alone (tools/gemm_time.py shapes) + ncu --set full of its first two launches (1 and 2 outputs, B MN-major)
mkdir -p gpurun_out
timeout 300 python tools/gemm_time.py 2>&1 | tail -4
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gemm_bf16_sm100" -s 2 -c 1 \
    -o gpurun_out/prof_f1 python tools/gemm_time.py > gpurun_out/ncu_f1.log 2>&1
echo "ncu rc=$?"
