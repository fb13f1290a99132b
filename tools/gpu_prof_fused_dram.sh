# DRAM bytes and L2 reduction misses of the fused backward (cfg3, rab on); one capture
mkdir -p gpurun_out
timeout 300 python tools/prof_attn.py 16 1 > /dev/null 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_red.sum,lts__t_sectors_srcunit_tex_op_red_lookup_miss.sum \
    --clock-control none -k regex:"fused" -c 1 --csv python tools/prof_attn.py 16 1 2>/dev/null | tail -6
