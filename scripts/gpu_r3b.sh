#!/bin/bash
# wide DTW kernel: grid sized by occupancy (4 CTAs per SM at S = 25)
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_appendix_b.py tests/test_gpu_search.py -x -q -k "wide or dtw_band or appendix or Wide" > gpurun_out/r3b_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r3b_tests.log
timeout 600 python scripts/appendix_b.py > gpurun_out/r3b_appendix_b.json 2> gpurun_out/r3b_appendix_b.err; echo "appb rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/r3b_appendix_b.json'))
print({k: '%.3g' % v['cells_per_s'] for k, v in d.items() if isinstance(v, dict) and 'cells_per_s' in v})" || tail -3 gpurun_out/r3b_appendix_b.err
timeout 600 python bench.py --config C3 --w 100 --no-cpu-baseline --steps 3 --warmup 3 > gpurun_out/r3b_C3w100.json 2> gpurun_out/r3b_C3w100.err
python -c "
import json; d=json.loads(open('gpurun_out/r3b_C3w100.json').read().strip().splitlines()[-1])
print('C3w100 ms %.1f' % d['ms_per_step'], {k: round(v,1) for k,v in d['stage_ms'].items()})"
