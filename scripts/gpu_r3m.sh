#!/bin/bash
# DTWLB_NO_ABANDON + full GPU suite + C5 bench
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/r3m_gpu_tests.log 2>&1; echo "gpu tests rc=$?"; tail -2 gpurun_out/r3m_gpu_tests.log
timeout 600 python bench.py --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/r3m_C5.json 2> gpurun_out/r3m_C5.err
python -c "
import json; d=json.loads(open('gpurun_out/r3m_C5.json').read().strip().splitlines()[-1])
print('C5 ms %.1f' % d['ms_per_step'], {k: round(v,1) for k,v in d['stage_ms'].items()})"
