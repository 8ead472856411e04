#!/bin/bash
# parameter sweep on C5 (plain runs): DTWLB_RANGES x DTWLB_RANGE_GROWTH
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
for RG in ${SWEEP:-2:8 3:8 4:8 3:16 4:4 5:4}; do
  R=${RG%%:*}; G=${RG##*:}
  DTWLB_RANGES=$R DTWLB_RANGE_GROWTH=$G python bench.py --no-cpu-baseline --steps 2 --warmup 1 ${BENCH_ARGS} > gpurun_out/sw_${R}_${G}.json 2>gpurun_out/sw.err
  python -c "
import json,sys
d=json.loads(open('gpurun_out/sw_${R}_${G}.json').read().strip().splitlines()[-1])
print('R=$R G=$G', round(d['ms_per_step'],1), {k: round(v,1) for k,v in d['stage_ms'].items()}, 'keogh', round(d['prune']['keogh_evaluated_frac'],4), 'imp', round(d['prune']['improved_evaluated_frac'],4), 'dtw', round(d['prune']['dtw_evaluated_frac'],5), 'cells', d['walk']['dtw_cells_computed'], 'rounds', d['walk']['walk_rounds'])
"
done
