#!/bin/bash
# Round-2 (session 3) validation + profile: GPU suite, smoke, bench lines, launch list, ncu of the gate
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/r3h_gpu_tests.log 2>&1; echo "gpu tests rc=$?"; tail -2 gpurun_out/r3h_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r3h_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r3h_smoke.log
timeout 900 python bench.py > gpurun_out/r3h_C5_bench.json 2> gpurun_out/r3h_C5_bench.err; echo "C5 rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/r3h_C5_bench.json').read().strip().splitlines()[-1])
print('C5 ms %.2f e2e %.4g frac %.3f' % (d['ms_per_step'], d['e2e']['value'], d['roofline']['frac']), d['step_ms'], {k: round(v,1) for k,v in d['stage_ms'].items()}, d['clocks'])"
for cfg in C4 C3 C5s1 C5s8; do
timeout 600 python bench.py --config $cfg --no-cpu-baseline > gpurun_out/r3h_${cfg}_bench.json 2> gpurun_out/r3h_${cfg}_bench.err
python -c "
import json; d=json.loads(open('gpurun_out/r3h_${cfg}_bench.json').read().strip().splitlines()[-1])
print('$cfg ms %.3f' % d['ms_per_step'], 'frac %.3f' % d['roofline']['frac'], d['roofline']['kernel'][:40])"
done
CMD="python bench.py --steps 1 --warmup 2 --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r3h_C5_launches.csv $CMD > gpurun_out/r3h_ncu_launch.log 2>&1; echo "launch list rc=$?"
python scripts/launch_summary.py gpurun_out/r3h_C5_launches.csv > gpurun_out/r3h_C5_launch_summary.txt 2>&1; head -14 gpurun_out/r3h_C5_launch_summary.txt
for KS in gate_sym_kernel:0; do
  K=${KS%%:*}; S=${KS##*:}
  R=gpurun_out/r3h_C5_${K}_$S
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s $S -c 1 -o $R $CMD > gpurun_out/r3h_ncu_${K}.log 2>&1
  echo "full $K rc=$?"
  python scripts/ncu_summary.py $R.ncu-rep > ${R}_ncu.txt 2>&1
  python scripts/ncu_lines.py $R.ncu-rep 40 > ${R}_lines.txt 2>&1
  ncu -i $R.ncu-rep --page raw --csv 2>/dev/null | python -c "
import csv,sys
r=list(csv.reader(sys.stdin)); h=r[0]; v=r[2]
d=dict(zip(h,v))
print('dram read', d.get('dram__bytes_read.sum'), 'write', d.get('dram__bytes_write.sum'), r[1][h.index('dram__bytes_read.sum')] if 'dram__bytes_read.sum' in h else '')" > ${R}_dram.txt
  rm -f $R.ncu-rep
  head -16 ${R}_ncu.txt; cat ${R}_dram.txt
done
