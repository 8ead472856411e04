#!/bin/bash
# ISA probes + launch list + full captures of the LB_Improved and DTW kernels (C5).
set -x
cd scripts && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/isa_probe isa_probe.cu && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/isa_probe2 isa_probe2.cu; cd ..
/tmp/isa_probe > gpurun_out/isa_probe.txt 2>&1
/tmp/isa_probe2 > gpurun_out/isa_probe2.txt 2>&1
CFG=${CFG:-C5}
CMD="python bench.py --config $CFG --steps 1 --warmup 1 --no-cpu-baseline"
$CMD > gpurun_out/p3_plain.json 2> gpurun_out/p3_plain.err || { echo "plain run failed"; tail gpurun_out/p3_plain.err; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/p3_launches.csv $CMD > gpurun_out/p3_ncu_launch.log 2>&1
for KS in ${CAPTURES:-improved_kernel:3 dtw_kernel:40}; do
  K=${KS%%:*}; S=${KS##*:}
  ncu --set full --clock-control none --import-source on -k regex:$K -s $S -c 1 -o gpurun_out/p3_${CFG}_${K}_$S $CMD > gpurun_out/p3_ncu_${K}.log 2>&1
  echo "full $K skip $S rc=$?"
done
