# ncu --set full (source) of the f1 SiLU GEMM via the test hook (tools/gemm_time.py)
set -x
mkdir -p gpurun_out
timeout 300 python tools/gemm_time.py > gpurun_out/gemm_time.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gemm_bf16" -s 2 -c 1 \
    -o gpurun_out/prof_gemm1 python tools/gemm_time.py > gpurun_out/ncu_gemm1.log 2>&1
echo "ncu rc=$?"
