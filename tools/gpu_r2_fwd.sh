# forward kernel iteration: parity (fwd + layer), timing, trace
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "fwd or layer or attn" > gpurun_out/r2f_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r2f_tests.log
timeout 600 python tools/attn_time.py > gpurun_out/r2f_time.log 2>&1; echo "time rc=$?"; grep "B=" gpurun_out/r2f_time.log
timeout 300 python tools/trace_fwd2.py 1 > gpurun_out/r2f_trace1.txt 2>&1; tail -8 gpurun_out/r2f_trace1.txt
