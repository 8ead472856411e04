#!/bin/bash
# tests + default bench + launch list, then bench variants given as env assignments in VARIANTS
bash scripts/gpu_quick.sh
for V in ${VARIANTS}; do
  env ${V//,/ } python bench.py --no-cpu-baseline --steps 2 --warmup 2 > gpurun_out/ab.json 2> gpurun_out/ab.err
  python -c "
import json; d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1])
print('$V', 'ms', round(d['ms_per_step'],1), {k: round(v,1) for k,v in d['stage_ms'].items()}, 'dtw_eval', d['walk']['dtw_evaluated'])"
done
