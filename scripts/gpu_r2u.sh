#!/bin/bash
# Round-2 re-entry check: GPU suite, smoke, C5 bench.
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/r2u_gpu_tests.log 2>&1; echo "gpu tests rc=$?"; tail -3 gpurun_out/r2u_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2u_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r2u_smoke.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/r2u_C5.json 2> gpurun_out/r2u_C5.err; echo "C5 rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/r2u_C5.json').read().strip().splitlines()[-1])
print('ms', d['ms_per_step'], 'e2e %.4g' % d['e2e']['value'], {k: round(v,1) for k,v in d['stage_ms'].items()})"
