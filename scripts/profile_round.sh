#!/bin/bash
# Round profile: plain bench (official defaults) -> other configs -> launch list -> ncu --set full
# of the hot kernels.  Outputs under gpurun_out/ (summaries are copied to profiles/).
TAG=${TAG:-r01}
CFG=${CFG:-C5}
python bench.py --config $CFG > gpurun_out/${TAG}_${CFG}_bench.json 2> gpurun_out/${TAG}_${CFG}_bench.err || { echo "bench failed"; tail gpurun_out/${TAG}_${CFG}_bench.err; exit 1; }
tail -1 gpurun_out/${TAG}_${CFG}_bench.json | cut -c1-300
for C in ${OTHER_CONFIGS}; do
  python bench.py --config $C --no-cpu-baseline > gpurun_out/${TAG}_${C}_bench.json 2> gpurun_out/${TAG}_${C}_bench.err; echo "$C rc=$?"
done
CMD="python bench.py --config $CFG --steps 1 --warmup 3 --no-cpu-baseline"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_${CFG}_launches.csv $CMD > gpurun_out/${TAG}_ncu_launch.log 2>&1
echo "launch list rc=$?"
for KS in ${CAPTURES:-improved_kernel:7 dtw4_kernel:100 keogh_tile_kernel:3}; do
  K=${KS%%:*}; S=${KS##*:}
  R=gpurun_out/${TAG}_${CFG}_${K}_$S
  ncu --set full --clock-control none --import-source on -k regex:$K -s $S -c 1 -o $R $CMD > gpurun_out/${TAG}_ncu_${K}_$S.log 2>&1
  echo "full $K skip $S rc=$?"
  # text summaries travel back; the reports themselves are large (gpurun_out <= 64 MiB)
  python scripts/ncu_summary.py $R.ncu-rep > ${R}_ncu.txt 2>&1
  python scripts/ncu_lines.py $R.ncu-rep 40 > ${R}_lines.txt 2>&1
  ncu -i $R.ncu-rep --page raw --csv > ${R}_raw.csv 2>/dev/null
  [ -n "$KEEP_REPS" ] || rm -f $R.ncu-rep
done
