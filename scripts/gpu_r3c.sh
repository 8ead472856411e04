#!/bin/bash
# select with half2 mask compares; wide kernel with 5 CTAs per SM at S = 25
timeout 900 python -m pytest tests/test_gpu_search.py tests/test_gpu_kernels.py tests/test_gpu_appendix_b.py tests/test_gpu_shards.py -x -q > gpurun_out/r3c_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r3c_tests.log
timeout 600 python scripts/appendix_b.py > gpurun_out/r3c_appendix_b.json 2> gpurun_out/r3c_appendix_b.err; echo "appb rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/r3c_appendix_b.json'))
print({k: '%.3g' % v['cells_per_s'] for k, v in d.items() if isinstance(v, dict) and 'cells_per_s' in v})" || tail -3 gpurun_out/r3c_appendix_b.err
timeout 600 python bench.py --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/r3c_C5.json 2> gpurun_out/r3c_C5.err
python -c "
import json; d=json.loads(open('gpurun_out/r3c_C5.json').read().strip().splitlines()[-1])
print('C5 ms %.1f' % d['ms_per_step'], {k: round(v,1) for k,v in d['stage_ms'].items()})"
CMD="python bench.py --config C5 --steps 1 --warmup 1 --no-cpu-baseline"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:select_mask8 --csv --log-file gpurun_out/r3c_select_launches.csv $CMD > /dev/null 2>&1; echo "ncu rc=$?"
grep -i "select_mask8" gpurun_out/r3c_select_launches.csv | head -4 | cut -c1-250
