#!/bin/bash
# select_mask8 with hoisted loads; ncu of the midpoint gate and the select kernel
timeout 900 python -m pytest tests/test_gpu_search.py tests/test_gpu_shards.py -x -q > gpurun_out/r2y_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r2y_tests.log
timeout 600 python bench.py --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/r2y_C5.json 2> gpurun_out/r2y_C5.err
python -c "
import json; d=json.loads(open('gpurun_out/r2y_C5.json').read().strip().splitlines()[-1])
print('C5 ms %.1f' % d['ms_per_step'], {k: round(v,1) for k,v in d['stage_ms'].items()})"
CMD="python bench.py --config C5 --steps 1 --warmup 1 --no-cpu-baseline"
for KS in gate_sym_kernel:1 select_mask8_kernel:1; do
  K=${KS%%:*}; S=${KS##*:}
  R=gpurun_out/r2y_C5_${K}_$S
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s $S -c 1 -o $R $CMD > gpurun_out/r2y_ncu_${K}.log 2>&1
  echo "full $K rc=$?"
  python scripts/ncu_summary.py $R.ncu-rep > ${R}_ncu.txt 2>&1
  python scripts/ncu_lines.py $R.ncu-rep 40 > ${R}_lines.txt 2>&1
  ncu -i $R.ncu-rep --page details --csv > ${R}_details.csv 2>/dev/null
  rm -f $R.ncu-rep
  head -22 ${R}_ncu.txt
done
