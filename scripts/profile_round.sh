#!/bin/bash
# Round profile: plain bench (official defaults) -> launch list -> ncu --set full of the
# hot kernels.  Outputs under gpurun_out/ (copy the summaries to profiles/).
TAG=${TAG:-r01}
CFG=${CFG:-C5}
python bench.py --config $CFG > gpurun_out/${TAG}_${CFG}_bench.json 2> gpurun_out/${TAG}_${CFG}_bench.err || { echo "bench failed"; tail gpurun_out/${TAG}_${CFG}_bench.err; exit 1; }
cat gpurun_out/${TAG}_${CFG}_bench.json
CMD="python bench.py --config $CFG --steps 1 --warmup 3 --no-cpu-baseline"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_${CFG}_launches.csv $CMD > gpurun_out/${TAG}_ncu_launch.log 2>&1
echo "launch list rc=$?"
for KS in ${CAPTURES:-improved_kernel:7 dtw4_kernel:100 keogh_tile_kernel:3}; do
  K=${KS%%:*}; S=${KS##*:}
  ncu --set full --clock-control none --import-source on -k regex:$K -s $S -c 1 -o gpurun_out/${TAG}_${CFG}_$K $CMD > gpurun_out/${TAG}_ncu_$K.log 2>&1
  echo "full $K skip $S rc=$?"
done
