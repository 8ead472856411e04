#!/bin/bash
# gate with half-chunk staging groups
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_search.py -x -q > gpurun_out/r2z_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r2z_tests.log
for cfg in C5 C4 C3; do
timeout 600 python bench.py --config $cfg --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/r2z_${cfg}.json 2> gpurun_out/r2z_${cfg}.err
python -c "
import json; d=json.loads(open('gpurun_out/r2z_${cfg}.json').read().strip().splitlines()[-1])
print('$cfg ms %.1f' % d['ms_per_step'], {k: round(v,1) for k,v in d['stage_ms'].items()})"
done
