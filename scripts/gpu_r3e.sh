#!/bin/bash
# per-reason warp stall breakdown (raw page) of the survivor and DTW kernels at C5
CMD="python bench.py --config C5 --steps 1 --warmup 1 --no-cpu-baseline"
for KS in improved_kernel:1 dtw4_kernel:13; do
  K=${KS%%:*}; S=${KS##*:}
  R=gpurun_out/r3e_C5_${K}_$S
  timeout 900 ncu --section WarpStateStats --section SchedulerStats --section InstructionStats --clock-control none -k regex:$K -s $S -c 1 -o $R $CMD > gpurun_out/r3e_ncu_${K}.log 2>&1
  echo "ws $K rc=$?"
  ncu -i $R.ncu-rep --page raw --csv > ${R}_raw.csv 2>/dev/null
  rm -f $R.ncu-rep
done
