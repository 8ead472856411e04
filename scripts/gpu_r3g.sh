#!/bin/bash
# gate with packed FADD2 midpoint elements
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_search.py -x -q -k "piecewise or C2 or reduced or switches or C1" > gpurun_out/r3g_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r3g_tests.log
for cfg in C5 C4 C3; do
timeout 600 python bench.py --config $cfg --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/r3g_${cfg}.json 2> gpurun_out/r3g_${cfg}.err
python -c "
import json; d=json.loads(open('gpurun_out/r3g_${cfg}.json').read().strip().splitlines()[-1])
print('$cfg ms %.1f' % d['ms_per_step'], 'gate %.1f' % d['stage_ms']['ms_keogh'])"
done
