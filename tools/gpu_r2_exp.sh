# time experiment builds (tools/build_exp.py) against the product build: attention fwd/bwd at cfg3
mkdir -p gpurun_out
echo "== product"; timeout 600 python tools/attn_time.py 2>&1 | grep "B="
for e in $(cat tools/exp/LIST); do echo "== exp $e"; UH_LIB=libuhstu_$e.so timeout 600 python tools/attn_time.py 2>&1 | grep "B="; done
if [ -n "$LAYER_TIME" ]; then
  for L in "" $(cat tools/exp/LIST); do echo "== layer ${L:-product}"; UH_LIB=${L:+libuhstu_$L.so} timeout 600 python tools/layer_time.py 2>&1 | grep "cfg3 layer"; done
fi
