# weak-scaling lines on N GPUs of one box: cfg3 and cfg4 (torchrun, NCCL)
N=$1
mkdir -p gpurun_out
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 \
    bench.py --gpus $N --steps 10 --warmup 3 > gpurun_out/bench_${N}gpu.json 2> gpurun_out/bench_${N}gpu.err
python -c "import json; d=json.loads(open('gpurun_out/bench_${N}gpu.json').read().strip().splitlines()[-1]); print('cfg3', $N, d['value'], d['ms_per_step'])"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29512 \
    bench.py --gpus $N --config cfg4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg4_${N}gpu.json 2> gpurun_out/bench_cfg4_${N}gpu.err
python -c "import json; d=json.loads(open('gpurun_out/bench_cfg4_${N}gpu.json').read().strip().splitlines()[-1]); print('cfg4', $N, d['value'], d['ms_per_step'])"
