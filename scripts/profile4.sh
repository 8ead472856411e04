#!/bin/bash
# tests + bench + ncu full captures of chosen launches (C5).
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
CMD="python bench.py --config ${CFG:-C5} --steps 1 --warmup 1 --no-cpu-baseline ${BENCH_ARGS}"
$CMD > gpurun_out/p4_plain.json 2> gpurun_out/p4_plain.err || { echo "plain run failed"; tail gpurun_out/p4_plain.err; exit 1; }
cat gpurun_out/p4_plain.json
for KS in ${CAPTURES:-improved_kernel:1}; do
  K=${KS%%:*}; S=${KS##*:}
  ncu --set full --clock-control none --import-source on -k regex:$K -s $S -c 1 -o gpurun_out/p4_${K}_$S $CMD > gpurun_out/p4_ncu_${K}.log 2>&1
  echo "full $K skip $S rc=$?"
done
