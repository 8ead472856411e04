#!/bin/bash
# Profile the bench command on one B200 (run under gpurun). Outputs in gpurun_out/.
# 1) plain run (must exit 0 first), 2) ncu launch list (device time per launch),
# 3) one `ncu --set full` capture per hot kernel.
CFG=${CFG:-C5}
CMD="python bench.py --config $CFG --steps 1 --warmup 3 --no-cpu-baseline"
$CMD > gpurun_out/prof_plain_$CFG.json 2> gpurun_out/prof_plain_$CFG.err || { echo "plain run failed"; tail gpurun_out/prof_plain_$CFG.err; exit 1; }
cat gpurun_out/prof_plain_$CFG.json
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$CFG.csv $CMD > gpurun_out/ncu_launch_$CFG.log 2>&1
echo "launch list rc=$?"
for K in ${KERNELS:-keogh_tile improved_kernel dtw_kernel}; do
  ncu --set full --clock-control none --import-source on -k regex:$K -s ${SKIP:-2} -c 1 -o gpurun_out/prof_${CFG}_$K $CMD > gpurun_out/ncu_${CFG}_$K.log 2>&1
  echo "full $K rc=$?"
done
