set -x
python tools/attn_time.py > gpurun_out/exp_base.log 2>&1; cat gpurun_out/exp_base.log | grep B=
cp paper_2602_16986_b200/lib/libuhstu_exp.so paper_2602_16986_b200/lib/libuhstu.so
python tools/attn_time.py > gpurun_out/exp_var.log 2>&1; cat gpurun_out/exp_var.log | grep B=
