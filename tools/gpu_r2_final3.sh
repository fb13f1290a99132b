# closing evidence (last): gpu_r2_final2.sh plus cfg5 and the MoT line
bash tools/gpu_r2_final2.sh
bash tools/gpu_r2_cfg5.sh
timeout 600 python bench.py --config mot --steps 10 --warmup 3 > gpurun_out/r2_mot.json 2> gpurun_out/r2_mot.err; echo "mot rc=$?"
