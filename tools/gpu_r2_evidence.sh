# round-2 evidence (outputs kept small: gpurun copies back <= 64 MiB): checked-build GPU suite,
# bench launch list, ncu --set full of every kernel of one cfg3 layer step (summarised on the box)
mkdir -p gpurun_out
UH_TEST_LIB=libuhstu_checked.so timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/r2e_checked_tests.log 2>&1; echo "checked tests rc=$?"; tail -2 gpurun_out/r2e_checked_tests.log
timeout 600 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2e_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1; echo "launch list rc=$?"
timeout 300 python tools/prof_layer.py 16 1 > /dev/null 2>&1 && \
timeout 1800 ncu --set full --clock-control none -c 40 -o /tmp/r2e_ncu_layer python tools/prof_layer.py 16 1 > gpurun_out/r2e_ncu_layer.log 2>&1; echo "ncu layer rc=$?"
python tools/ncu_summary.py /tmp/r2e_ncu_layer.ncu-rep gpurun_out/r2e_ncu_layer.json > gpurun_out/r2e_ncu_layer.txt 2>&1; echo "summary rc=$?"
ncu -i /tmp/r2e_ncu_layer.ncu-rep --page raw --csv > /tmp/raw.csv 2>/dev/null; gzip -c /tmp/raw.csv > gpurun_out/r2e_ncu_layer_raw.csv.gz; ls -la gpurun_out
