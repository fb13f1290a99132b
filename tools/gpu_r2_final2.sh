# round-2 closing evidence: smoke, full GPU suite (product), then tools/gpu_r2_final.sh
mkdir -p gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/rf_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/rf_smoke.log
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/rf_gpu_tests.log 2>&1; echo "gpu tests rc=$?"; tail -2 gpurun_out/rf_gpu_tests.log
bash tools/gpu_r2_final.sh
