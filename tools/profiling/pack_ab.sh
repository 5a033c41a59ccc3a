# A/B of the forward tile packing (BSA_FWD_PACK / BSA_FWD_ORDER) on the BASELINE workloads and the dense path
O=gpurun_out/pk3; mkdir -p $O
for v in "BSA_FWD_PACK=0" "BSA_FWD_ORDER=small" "BSA_FWD_PACK=16 BSA_FWD_ORDER=small"; do
  for c in wan1.3b_32k wan14b_75k long_147k; do
    env $v timeout 300 python tools/profiling/time_attn.py $c 5 >> $O/t.txt 2>&1; echo "$v $c" >> $O/t.txt
  done
done
