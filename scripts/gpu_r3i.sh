#!/bin/bash
# DTW: odd-step packed FADD2 differences
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_search.py tests/test_gpu_colcasc.py -x -q > gpurun_out/r3i_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r3i_tests.log
for cfg in C5 C2p1; do
timeout 600 python bench.py --config $cfg --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/r3i_${cfg}.json 2> gpurun_out/r3i_${cfg}.err
python -c "
import json; d=json.loads(open('gpurun_out/r3i_${cfg}.json').read().strip().splitlines()[-1])
print('$cfg ms %.1f' % d['ms_per_step'], 'dtw_kernel %.2f cells %.4g frac %.3f' % (d['stage_ms']['ms_dtw_kernel'], d['walk']['dtw_cells_computed'], d['roofline']['dtw_kernel']['frac']))"
done
