# NEXT-3 LBSL: GPU parity + timing + ncu of the gather kernel; outputs under gpurun_out/
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
#timeout 600 python -m pytest tests/test_gpu_lbsl.py tests/test_lbsl_native.py -x -q 2>&1 | tail -5 | tee gpurun_out/lbsl_tests.log
timeout 300 python tools/lbsl_time.py 2>&1 | tail -3 | tee gpurun_out/lbsl_time.log
timeout 600 ncu --set full --clock-control none -k regex:gather_rows_k -c 1 --csv --page raw \
    python tools/lbsl_time.py > gpurun_out/lbsl_ncu_raw.csv 2> gpurun_out/lbsl_ncu.err
echo "ncu rc=$?"
