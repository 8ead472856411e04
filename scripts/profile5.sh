#!/bin/bash
# tests + bench + launch list + ncu full captures (C5).
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
CMD="python bench.py --config ${CFG:-C5} --steps 1 --warmup 1 --no-cpu-baseline ${BENCH_ARGS}"
$CMD > gpurun_out/p5_plain.json 2> gpurun_out/p5_plain.err || { echo "plain run failed"; tail gpurun_out/p5_plain.err; exit 1; }
cat gpurun_out/p5_plain.json
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/p5_launches.csv $CMD > gpurun_out/p5_ncu_launch.log 2>&1
echo "launch list rc=$?"
for KS in ${CAPTURES:-improved_kernel:1 dtw4_kernel:30}; do
  K=${KS%%:*}; S=${KS##*:}
  ncu --set full --clock-control none --import-source on -k regex:$K -s $S -c 1 -o gpurun_out/p5_${K}_$S $CMD > gpurun_out/p5_ncu_${K}.log 2>&1
  echo "full $K skip $S rc=$?"
done
