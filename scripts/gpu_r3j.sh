#!/bin/bash
# survivor kernel with packed FADD2 element pairs
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_search.py -x -q > gpurun_out/r3j_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r3j_tests.log
for cfg in C5 C4 C3; do
timeout 600 python bench.py --config $cfg --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/r3j_${cfg}.json 2> gpurun_out/r3j_${cfg}.err
python -c "
import json; d=json.loads(open('gpurun_out/r3j_${cfg}.json').read().strip().splitlines()[-1])
print('$cfg ms %.1f' % d['ms_per_step'], 'surv %.2f' % d['stage_ms']['ms_survivor_kernel'], 'frac_mix %.3f' % d['roofline']['survivor_kernel']['frac_of_mix_peak'])"
done
