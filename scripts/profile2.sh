#!/bin/bash
# Full ncu captures of selected launches (after a plain run that exited 0).
CFG=${CFG:-C5}
CMD="python bench.py --config $CFG --steps 1 --warmup 1 --no-cpu-baseline"
$CMD > gpurun_out/p2_plain.json 2> gpurun_out/p2_plain.err || { echo "plain run failed"; tail gpurun_out/p2_plain.err; exit 1; }
cat gpurun_out/p2_plain.json
# kernel:skip pairs
for KS in ${CAPTURES:-improved_kernel:5 dtw_kernel:60 select_mask:3}; do
  K=${KS%%:*}; S=${KS##*:}
  ncu --set full --clock-control none --import-source on -k regex:$K -s $S -c 1 -o gpurun_out/p2_${CFG}_${K}_$S $CMD > gpurun_out/p2_ncu_${K}.log 2>&1
  echo "full $K skip $S rc=$?"
done
