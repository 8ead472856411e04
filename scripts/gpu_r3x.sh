#!/bin/bash
# A/B of a survivor-kernel change: the search/schedule/shard GPU tests, then the C5 bench line
timeout 1200 python -m pytest tests/test_gpu_search.py tests/test_gpu_colcasc.py tests/test_gpu_shards.py -m gpu -x -q > gpurun_out/r3x_gpu_tests.log 2>&1; echo "gpu tests rc=$?"; tail -2 gpurun_out/r3x_gpu_tests.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r3x_C5_bench.json 2> gpurun_out/r3x_C5_bench.err; echo "C5 rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/r3x_C5_bench.json').read().strip().splitlines()[-1])
s=d['stage_ms']; print('C5 ms %.2f' % d['ms_per_step'], 'gate %.1f surv %.1f dtwk %.1f improved-stage %.1f' % (s['ms_keogh'], s['ms_survivor_kernel'], s['ms_dtw_kernel'], s['ms_improved']), d['step_ms'])"
