#!/bin/bash
# Round-2 final profile: launch list of the C5 bench + ncu --set full of the hot kernels.
CMD="python bench.py --steps 1 --warmup 2 --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2r_C5_launches.csv $CMD > gpurun_out/r2r_ncu_launch.log 2>&1; echo "launch list rc=$?"
python scripts/launch_summary.py gpurun_out/r2r_C5_launches.csv > gpurun_out/r2r_C5_launch_summary.txt 2>&1; head -30 gpurun_out/r2r_C5_launch_summary.txt
for KS in improved_kernel:1 dtw4_kernel:13 gate_sym_kernel:0; do
  K=${KS%%:*}; S=${KS##*:}
  R=gpurun_out/r2r_C5_${K}_$S
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s $S -c 1 -o $R $CMD > gpurun_out/r2r_ncu_${K}.log 2>&1
  echo "full $K rc=$?"
  python scripts/ncu_summary.py $R.ncu-rep > ${R}_ncu.txt 2>&1
  python scripts/ncu_lines.py $R.ncu-rep 40 > ${R}_lines.txt 2>&1
  head -16 ${R}_ncu.txt
done
