# source-level ncu (warp-stall samples per SASS / CUDA line) of the fused attention backward and
# the forward at cfg3, rab on; summarised on the box (the .ncu-rep itself stays there)
mkdir -p gpurun_out
timeout 300 python tools/prof_attn.py 16 1 > /dev/null 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"attn_bwd_fused|attn_fwd_sm100" -c 2 \
    -o /tmp/r2src python tools/prof_attn.py 16 1 > gpurun_out/r2src_ncu.log 2>&1
echo "ncu rc=$?"; tail -2 gpurun_out/r2src_ncu.log
ncu -i /tmp/r2src.ncu-rep --page source --csv --print-source sass > /tmp/src_sass.csv 2>/dev/null
ncu -i /tmp/r2src.ncu-rep --page source --csv --print-source cuda > /tmp/src_cuda.csv 2>/dev/null
python tools/ncu_src.py /tmp/src_sass.csv attn_bwd_fused 80 > gpurun_out/r2src_bwd_sass.txt 2>&1
python tools/ncu_src.py /tmp/src_sass.csv attn_fwd_sm100 60 > gpurun_out/r2src_fwd_sass.txt 2>&1
python tools/ncu_src.py /tmp/src_cuda.csv attn_bwd_fused 60 > gpurun_out/r2src_bwd_cuda.txt 2>&1
python tools/ncu_src.py /tmp/src_cuda.csv attn_fwd_sm100 50 > gpurun_out/r2src_fwd_cuda.txt 2>&1
gzip -c /tmp/src_sass.csv > gpurun_out/r2src_sass.csv.gz; gzip -c /tmp/src_cuda.csv > gpurun_out/r2src_cuda.csv.gz
ls -la gpurun_out | tail -8; head -5 gpurun_out/r2src_bwd_cuda.txt
