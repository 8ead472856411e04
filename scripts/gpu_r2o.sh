#!/bin/bash
timeout 1800 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_appendix_b.py tests/test_gpu_search.py -x -q -k "wide or dtw or appendix or band" > gpurun_out/r2o_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r2o_tests.log
for KW in 8 4; do
  DTWLB_WIDE_KW=$KW timeout 600 python bench.py --config C3 --w 100 --no-cpu-baseline --steps 5 > gpurun_out/r2o_C3w100_kw$KW.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/r2o_C3w100_kw$KW.json').read().strip().splitlines()[-1])
print('C3w100 KW=$KW ms', round(d['ms_per_step'],2), {k: round(v,2) for k,v in d['stage_ms'].items() if k in ('ms_improved','ms_dtw','ms_dtw_kernel')}, d['walk']['dtw_cells_computed'])"
  DTWLB_WIDE_KW=$KW timeout 300 python scripts/appendix_b.py 100000 --no-oracle > gpurun_out/r2o_appb_kw$KW.json 2>&1
  python -c "
import json; d=json.load(open('gpurun_out/r2o_appb_kw$KW.json')); print('AppB KW=$KW', {k:(round(v['violation_frac'],4), '%.3g cells/s' % v['cells_per_s'], round(v['seconds']*1e3,3)) for k,v in d.items()})"
done
for C in C5 C3 C4; do
  timeout 900 python bench.py --config $C --no-cpu-baseline > gpurun_out/r2o_$C.json 2> gpurun_out/r2o_$C.err; echo "$C rc=$?"
  python -c "
import json; d=json.loads(open('gpurun_out/r2o_$C.json').read().strip().splitlines()[-1])
print('$C ms', d['ms_per_step'], 'steps', d['step_ms']); print({k: round(v,2) for k,v in d['stage_ms'].items()})"
done
