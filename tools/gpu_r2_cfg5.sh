# cfg5 (inference, BASELINE configs[4]): batch filling the GPU, L in {4096, 16384, 65536}
mkdir -p gpurun_out
for L in 4096 16384 65536; do
  timeout 1200 python bench.py --config cfg5 --seq-len $L --tokens 0 --steps 3 --warmup 3 > gpurun_out/r2_cfg5_L$L.json 2> gpurun_out/r2_cfg5_L$L.err
  echo "L=$L rc=$?"; head -c 1500 gpurun_out/r2_cfg5_L$L.json; echo; tail -2 gpurun_out/r2_cfg5_L$L.err
done
