# round-2 final evidence (outputs small: gpurun copies back <= 64 MiB): bench line, launch list,
# ncu --set full of the attention kernels and of every kernel of one layer step (summarised on
# the box), FP8 vs bf16 projection timings + ncu, checked-build GPU suite, attention timings
mkdir -p gpurun_out
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/rf_bench.json 2> gpurun_out/rf_bench.err; echo "bench rc=$?"
ATTN_TIME_CAUSAL_RAB=1 ATTN_TIME_SPLIT=1 timeout 600 python tools/attn_time.py 2>&1 | grep "B=" > gpurun_out/rf_attn_time.log; cat gpurun_out/rf_attn_time.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/rf_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1; echo "launch list rc=$?"
timeout 1800 ncu --set full --clock-control none -c 40 -o /tmp/rf_layer python tools/prof_layer.py 16 1 > gpurun_out/rf_ncu_layer.log 2>&1; echo "ncu layer rc=$?"
python tools/ncu_summary.py /tmp/rf_layer.ncu-rep gpurun_out/rf_ncu_layer.json > /dev/null 2>&1
ncu -i /tmp/rf_layer.ncu-rep --page raw --csv > /tmp/rf_raw.csv 2>/dev/null; gzip -c /tmp/rf_raw.csv > gpurun_out/rf_ncu_layer_raw.csv.gz
timeout 900 ncu --set full --clock-control none -k regex:"attn_bwd_fused|dq_finish|attn_fwd_sm100" -c 3 -o /tmp/rf_attn python tools/prof_attn.py 16 1 > gpurun_out/rf_ncu_attn.log 2>&1; echo "ncu attn rc=$?"
python tools/ncu_summary.py /tmp/rf_attn.ncu-rep gpurun_out/rf_ncu_attn.json > /dev/null 2>&1
ncu -i /tmp/rf_attn.ncu-rep --page raw --csv > /tmp/rf_attn_raw.csv 2>/dev/null; gzip -c /tmp/rf_attn_raw.csv > gpurun_out/rf_ncu_attn_raw.csv.gz
timeout 600 python tools/fp8_time.py > gpurun_out/rf_fp8_time.log 2>&1; tail -9 gpurun_out/rf_fp8_time.log
timeout 900 ncu --set full --clock-control none -k regex:gemm_bf16_sm100 -c 4 -o /tmp/rf_gemm python tools/gemm_once.py > gpurun_out/rf_ncu_gemm.log 2>&1; echo "ncu gemm rc=$?"
ncu -i /tmp/rf_gemm.ncu-rep --page raw --csv > /tmp/rf_gemm_raw.csv 2>/dev/null; gzip -c /tmp/rf_gemm_raw.csv > gpurun_out/rf_ncu_gemm_raw.csv.gz
UH_TEST_LIB=libuhstu_checked.so timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/rf_checked_tests.log 2>&1; echo "checked tests rc=$?"; tail -2 gpurun_out/rf_checked_tests.log
ls -la gpurun_out | tail -20
