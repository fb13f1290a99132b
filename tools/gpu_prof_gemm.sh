# ncu --set full of the first f1 (SiLU) GEMM launch inside the bench
set -x
mkdir -p gpurun_out
timeout 600 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_short.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gemm_bf16_sm100" -s ${SKIP:-0} -c ${COUNT:-6} \
    -o gpurun_out/prof_gemm python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_gemm.log 2>&1
echo "ncu rc=$?"
