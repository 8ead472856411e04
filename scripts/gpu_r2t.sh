#!/bin/bash
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/r2t_gpu_tests.log 2>&1; echo "gpu tests rc=$?"; tail -3 gpurun_out/r2t_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2t_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r2t_smoke.log
DTWLB_LIB=$PWD/paper_0811_3301_b200/libdtwlb_checked.so timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/r2t_checked_tests.log 2>&1
echo "checked gpu tests rc=$?"; tail -2 gpurun_out/r2t_checked_tests.log
timeout 900 python bench.py > gpurun_out/r2t_C5.json 2> gpurun_out/r2t_C5.err; echo "C5 rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/r2t_C5.json').read().strip().splitlines()[-1])
print('ms', d['ms_per_step'], 'e2e %.4g' % d['e2e']['value'], 'steps', d['step_ms'])"
