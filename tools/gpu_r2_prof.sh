# round 2: compute-sanitizer logs on the small ragged cases, ncu --set full of the attention
# kernels (cfg3, rab on) and of every kernel of one cfg3 layer step
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2p_smi.txt
timeout 300 python tools/sanitize_case.py > gpurun_out/r2p_plain.log 2>&1; echo "plain rc=$?"; tail -5 gpurun_out/r2p_plain.log
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 40 python tools/sanitize_case.py > gpurun_out/r2p_san_$tool.log 2>&1
  echo "$tool rc=$?"; tail -4 gpurun_out/r2p_san_$tool.log
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"attn_fwd|attn_bwd_fused|dq_finish" -c 3 \
   -o gpurun_out/r2p_ncu_attn python tools/prof_attn.py 16 1 > gpurun_out/r2p_ncu_attn.log 2>&1; echo "ncu attn rc=$?"
timeout 1500 ncu --set full --clock-control none -c 24 -o gpurun_out/r2p_ncu_layer python tools/prof_layer.py 16 1 \
   > gpurun_out/r2p_ncu_layer.log 2>&1; echo "ncu layer rc=$?"
ls -la gpurun_out/
