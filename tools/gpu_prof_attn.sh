set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 300 python tools/prof_attn.py 2 ${RAB:-0} > gpurun_out/prof_plain.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on \
    -k regex:"attn_" -s 3 -c 3 -o gpurun_out/prof_attn \
    python tools/prof_attn.py 2 ${RAB:-0} > gpurun_out/ncu_attn.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/ncu_attn.log
