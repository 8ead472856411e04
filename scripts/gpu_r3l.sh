#!/bin/bash
# DTW: row -1 band copied from a shared-memory template (no 2w+2 register moves per start)
timeout 1200 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_search.py tests/test_gpu_colcasc.py tests/test_gpu_shards.py -x -q > gpurun_out/r3l_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r3l_tests.log
for cfg in C5 C4 C3; do
timeout 600 python bench.py --config $cfg --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/r3l_${cfg}.json 2> gpurun_out/r3l_${cfg}.err
python -c "
import json; d=json.loads(open('gpurun_out/r3l_${cfg}.json').read().strip().splitlines()[-1])
print('$cfg ms %.1f' % d['ms_per_step'], 'dtw_kernel %.2f frac %.3f' % (d['stage_ms']['ms_dtw_kernel'], d['roofline']['dtw_kernel']['frac']))"
done
