# cfg4 (18-layer stack) and cfg5 (inference) lines on one B200
mkdir -p gpurun_out
timeout 900 python bench.py --config cfg4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err
python -c "import json; d=json.load(open('gpurun_out/bench_cfg4.json')); print('cfg4', d['value'], d['ms_per_step'])"
for L in 4096 16384 65536; do
  timeout 900 python bench.py --config cfg5 --seq-len $L --steps 3 --warmup 1 --no-cpu-baseline > gpurun_out/bench_cfg5_$L.json 2> gpurun_out/bench_cfg5_$L.err
  python -c "import json; d=json.load(open('gpurun_out/bench_cfg5_$L.json')); print('cfg5', $L, d['value'], d['ms_per_step'], d.get('gpu_launches_per_step'))"
done
