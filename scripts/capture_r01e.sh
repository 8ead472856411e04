TAG=r01e; CFG=C5
CMD="python bench.py --config $CFG --steps 1 --warmup 3 --no-cpu-baseline"
for KS in improved_kernel:7 dtw4_kernel:33 keogh_tile_kernel:6 keogh_tile_kernel:7; do
  K=${KS%%:*}; S=${KS##*:}
  R=gpurun_out/${TAG}_${CFG}_${K}_$S
  ncu --set full --clock-control none --import-source on -k regex:$K -s $S -c 1 -o $R $CMD > gpurun_out/${TAG}_ncu_${K}_$S.log 2>&1
  echo "full $K skip $S rc=$?"
  python scripts/ncu_summary.py $R.ncu-rep > ${R}_ncu.txt 2>&1
  python scripts/ncu_lines.py $R.ncu-rep 40 > ${R}_lines.txt 2>&1
  ncu -i $R.ncu-rep --page raw --csv > ${R}_raw.csv 2>/dev/null
  rm -f $R.ncu-rep
done
