#!/bin/bash
# warp-state (stall reason) breakdown of the survivor and DTW kernels at C5
CMD="python bench.py --config C5 --steps 1 --warmup 1 --no-cpu-baseline"
for KS in improved_kernel:1 dtw4_kernel:13; do
  K=${KS%%:*}; S=${KS##*:}
  R=gpurun_out/r3d_C5_${K}_$S
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s $S -c 1 -o $R $CMD > gpurun_out/r3d_ncu_${K}.log 2>&1
  echo "full $K rc=$?"
  ncu -i $R.ncu-rep --page details --csv > ${R}_details.csv 2>/dev/null
  python scripts/ncu_summary.py $R.ncu-rep > ${R}_ncu.txt 2>&1
  rm -f $R.ncu-rep
  grep -i "stall\|throttle" ${R}_details.csv | cut -c1-200 | head -40
done
