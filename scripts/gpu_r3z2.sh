#!/bin/bash
# per-instruction stall samples of the largest DTW walk launch (SASS source page of one ncu capture)
CMD="python bench.py --config C5 --steps 1 --warmup 3 --no-cpu-baseline"
R=gpurun_out/r02zl_C5_dtw4_kernel_10
ncu --set full --clock-control none --import-source on -k regex:dtw4_kernel -s 10 -c 1 -o $R $CMD > gpurun_out/r02zl_ncu_dtw.log 2>&1; echo "ncu rc=$?"
ncu -i $R.ncu-rep --page source --csv --print-source sass > ${R}_sass.csv 2> gpurun_out/r02zl_sass_dtw.err; echo "sass rc=$?"; ls -la ${R}_sass.csv
rm -f $R.ncu-rep
