# round-end measurements on one B200: GPU tests, smoke, bench + launch list, cfg4, cfg5 lines
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
bash tools/gpu_bench.sh > /dev/null 2>&1
python -c "import json; d=json.load(open('gpurun_out/bench.json')); print('cfg3', d['value'], d['ms_per_step'], d['e2e']['value'], d['roofline']['frac'], d['clocks'])"
timeout 900 python bench.py --config cfg4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err
python -c "import json; d=json.load(open('gpurun_out/bench_cfg4.json')); print('cfg4', d['value'], d['ms_per_step'])"
for L in 16384 32768 65536; do
  timeout 900 python bench.py --config cfg5 --seq-len $L --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg5_$L.json 2> gpurun_out/bench_cfg5_$L.err
  python -c "import json; d=json.load(open('gpurun_out/bench_cfg5_$L.json')); print('cfg5', $L, d['value'], d['ms_per_step'])"
done
