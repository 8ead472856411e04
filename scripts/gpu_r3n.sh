#!/bin/bash
# final captures: launch list of the C5 bench, ncu --set full of the DTW walk's largest launch and the survivor kernel
CMD="python bench.py --steps 1 --warmup 2 --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r3n_C5_launches.csv $CMD > gpurun_out/r3n_ncu_launch.log 2>&1; echo "launch list rc=$?"
python scripts/launch_summary.py gpurun_out/r3n_C5_launches.csv > gpurun_out/r3n_C5_launch_summary.txt 2>&1; head -8 gpurun_out/r3n_C5_launch_summary.txt
for KS in dtw4_kernel:13 improved_kernel:1; do
  K=${KS%%:*}; S=${KS##*:}
  R=gpurun_out/r3n_C5_${K}_$S
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s $S -c 1 -o $R $CMD > gpurun_out/r3n_ncu_${K}.log 2>&1
  echo "full $K rc=$?"
  python scripts/ncu_summary.py $R.ncu-rep > ${R}_ncu.txt 2>&1
  python scripts/ncu_lines.py $R.ncu-rep 40 > ${R}_lines.txt 2>&1
  ncu -i $R.ncu-rep --page raw --csv 2>/dev/null | python -c "
import csv,sys
r=list(csv.reader(sys.stdin)); h=r[0]; u=r[1]; v=r[2]
for m in ('dram__bytes_read.sum','dram__bytes_write.sum','gpu__time_duration.sum'):
    if m in h: i=h.index(m); print(m, v[i], u[i])" > ${R}_dram.txt
  rm -f $R.ncu-rep
  head -16 ${R}_ncu.txt; cat ${R}_dram.txt
done
