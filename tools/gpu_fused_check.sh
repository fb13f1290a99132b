# fused attention backward: parity first (hard timeouts), then bench both backward variants
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "attn_bwd" -x 2>&1 | tail -15
rc=${PIPESTATUS[0]}
echo "attn_bwd rc=$rc"
[ "$rc" = "0" ] || exit 1
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -5
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_fused.json 2> gpurun_out/bench_fused.err
echo "fused bench rc=$?"; cat gpurun_out/bench_fused.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('fused', d['value'], d['ms_per_step'], d.get('attn'))"
UH_ATTN_BWD=split timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_split.json 2> gpurun_out/bench_split.err
cat gpurun_out/bench_split.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('split', d['value'], d['ms_per_step'], d.get('attn'))"
