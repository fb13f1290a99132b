set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -5
timeout 1200 python -m pytest tests -m gpu -q --timeout 300 --timeout-method=thread -p no:cacheprovider -rf > gpurun_out/pytest.log 2>&1
echo "pytest rc=$?"
tail -60 gpurun_out/pytest.log
