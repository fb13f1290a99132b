# attention kernels timed alone (cfg3, rab on) with the default and variant libraries:
#   attn_time_lib.sh NAME...   (paper_2602_16986_b200/lib/libuhstu_NAME.so)
L=paper_2602_16986_b200/lib
echo "== default"; timeout 300 python tools/attn_time_lib.py $L/libuhstu.so 16 1 2>&1 | grep "B=16"
for n in "$@"; do
  echo "== $n"; timeout 300 python tools/attn_time_lib.py $L/libuhstu_$n.so 16 1 2>&1 | grep "B=16"
done
