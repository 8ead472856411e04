#!/bin/bash
# A/B of env switches on the C5 bench (plain runs): AB_VARS="A=1 B=1,C=2" -> one run per entry
# (comma = several variables at once) plus a baseline.
run() { python bench.py --no-cpu-baseline --steps 2 --warmup 3 ${BENCH_ARGS} > gpurun_out/ab.json 2> gpurun_out/ab.err;
  python -c "
import json; d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1])
print('$1', 'ms', round(d['ms_per_step'],1), {k: round(v,1) for k,v in d['stage_ms'].items()}, 'cells', d['walk']['dtw_cells_computed'])"; }
run base
for v in ${AB_VARS}; do env $(echo $v | tr , " ") bash -c "$(declare -f run); run $v"; done
