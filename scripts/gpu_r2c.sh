#!/bin/bash
# Round-2 checkpoint c: compute-sanitizer tier (memcheck / racecheck / synccheck on the small
# oracle-checked workloads, release and DTWLB_CHECKED builds), the checked build under the GPU
# suite, and ncu captures of the largest DTW walk launch and the fused gate for the traffic table.
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 $CS --tool $tool --error-exitcode 9 --target-processes all python scripts/sanitize_case.py > gpurun_out/r2c_sanitize_$tool.log 2>&1
  echo "$tool rc=$?"; tail -3 gpurun_out/r2c_sanitize_$tool.log
done
DTWLB_LIB=$PWD/paper_0811_3301_b200/libdtwlb_checked.so timeout 1200 $CS --tool memcheck --error-exitcode 9 python scripts/sanitize_case.py > gpurun_out/r2c_sanitize_checked_memcheck.log 2>&1
echo "checked memcheck rc=$?"; tail -2 gpurun_out/r2c_sanitize_checked_memcheck.log
DTWLB_LIB=$PWD/paper_0811_3301_b200/libdtwlb_checked.so timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2c_checked_tests.log 2>&1
echo "checked gpu tests rc=$?"; tail -2 gpurun_out/r2c_checked_tests.log
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline"
for KS in dtw4_kernel:13 gate_sym_kernel:0 select_mask8:1; do
  K=${KS%%:*}; S=${KS##*:}
  R=gpurun_out/r2c_C5_${K}_$S
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s $S -c 1 -o $R $CMD > gpurun_out/r2c_ncu_${K}.log 2>&1
  echo "full $K rc=$?"
  python scripts/ncu_summary.py $R.ncu-rep > ${R}_ncu.txt 2>&1
  python scripts/ncu_lines.py $R.ncu-rep 40 > ${R}_lines.txt 2>&1
done
