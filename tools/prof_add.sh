set -u
mkdir -p gpurun_out
for W in c2 c5; do for OP in add sub_l2; do
  PROFILE_ONLY=$OP timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_add -c 2 -f -o /tmp/p_${W}_$OP python tools/profile_ops.py $W > gpurun_out/ncu_${W}_$OP.log 2>&1
  ncu -i /tmp/p_${W}_$OP.ncu-rep --page details --csv > gpurun_out/det_${W}_$OP.csv 2>/dev/null
  ncu -i /tmp/p_${W}_$OP.ncu-rep --page raw --csv > gpurun_out/raw_${W}_$OP.csv 2>/dev/null
  ncu -i /tmp/p_${W}_$OP.ncu-rep --page source --csv --print-source sass > gpurun_out/src_${W}_$OP.csv 2>/dev/null
done; done
ls -la gpurun_out
