# attention-only timing sweep (fast iteration); outputs gpurun_out/attn_*.json
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 600 python tools/attn_time.py > gpurun_out/attn_time.log 2>&1
echo "rc=$?"; cat gpurun_out/attn_time.log
