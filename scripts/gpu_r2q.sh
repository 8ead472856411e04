#!/bin/bash
timeout 1200 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_appendix_b.py tests/test_gpu_search.py -x -q -k "wide or eight or appendix or host or band" > gpurun_out/r2q_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r2q_tests.log
timeout 300 python scripts/appendix_b.py 100000 --no-oracle > gpurun_out/r2q_appb.json 2>&1
python -c "
import json; d=json.load(open('gpurun_out/r2q_appb.json')); print('AppB', {k:(round(v['violation_frac'],4), '%.3g cells/s' % v['cells_per_s'], round(v['seconds']*1e3,3)) for k,v in d.items()})"
timeout 600 python bench.py --config C3 --w 100 --no-cpu-baseline --steps 5 > gpurun_out/r2q_C3w100.json 2>/dev/null
python -c "
import json; d=json.loads(open('gpurun_out/r2q_C3w100.json').read().strip().splitlines()[-1])
print('C3w100 ms', round(d['ms_per_step'],2), {k: round(v,2) for k,v in d['stage_ms'].items() if k in ('ms_improved','ms_dtw','ms_dtw_kernel')})"
