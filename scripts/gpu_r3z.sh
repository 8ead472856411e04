#!/bin/bash
# per-instruction stall samples of the survivor kernel (SASS source page of one ncu capture)
CMD="python bench.py --config C5 --steps 1 --warmup 3 --no-cpu-baseline"
R=gpurun_out/r02zl_C5_improved_kernel_1
ncu --set full --clock-control none --import-source on -k regex:improved_kernel -s 1 -c 1 -o $R $CMD > gpurun_out/r02zl_ncu.log 2>&1; echo "ncu rc=$?"
ncu -i $R.ncu-rep --page source --csv --print-source sass > ${R}_sass.csv 2> gpurun_out/r02zl_sass.err; echo "sass rc=$?"; ls -la ${R}_sass.csv
head -c 600 ${R}_sass.csv
rm -f $R.ncu-rep
