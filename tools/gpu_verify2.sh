# re-entry verification on NG (default 2) B200s: the torchrun bench line (NCCL grad all-reduce)
mkdir -p gpurun_out
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node ${NG:-2} --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus ${NG:-2} --steps 10 --warmup 3 > gpurun_out/verify_bench_${NG:-2}gpu.json 2> gpurun_out/verify_bench_${NG:-2}gpu.err
tail -c 600 gpurun_out/verify_bench_${NG:-2}gpu.json
