# DRAM / L2 traffic of the attention kernels at cfg3 scale (B, RAB env)
set -x
mkdir -p gpurun_out
timeout 300 python tools/prof_attn.py ${B:-16} ${RAB:-1} > gpurun_out/prof_plain.log 2>&1 && \
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,lts__t_sector_hit_rate.pct,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_tc.avg.pct_of_peak_sustained_elapsed \
    --clock-control none -k regex:"attn_" -s 3 -c 3 --csv python tools/prof_attn.py ${B:-16} ${RAB:-1} > gpurun_out/ncu_mem.csv 2> gpurun_out/ncu_mem.err
echo "ncu rc=$?"
