#!/bin/bash
# final tree: ncu launch list of the bench command (shares of the step per kernel)
CMD="python bench.py --config C5 --steps 1 --warmup 3 --no-cpu-baseline"
$CMD > gpurun_out/r02zm_plain.json 2> gpurun_out/r02zm_plain.err; echo "plain rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02zm_C5_launches.csv $CMD > gpurun_out/r02zm_ncu_launch.log 2>&1; echo "launch list rc=$?"
python scripts/launch_summary.py gpurun_out/r02zm_C5_launches.csv 6 > gpurun_out/r02zm_C5_launch_summary.txt 2>&1; head -8 gpurun_out/r02zm_C5_launch_summary.txt
