#!/bin/bash
# Launch list of the default C5 run, then the paper's comparison (Alg. 2 = LB_Keogh only vs
# Alg. 3 = LB_Keogh + LB_Improved) and the pre-filter ablation, per config (plain runs).
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/q_launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
python scripts/launch_summary.py gpurun_out/q_launches.csv 4 2>/dev/null | head -8
for C in ${CONFIGS:-C5 C4 C3 C2p1 C2p2}; do
  for M in "" "--keogh-only" "--no-prefilter" "--keogh-only --no-prefilter"; do
    python bench.py --config $C --no-cpu-baseline --steps 2 --warmup 3 $M > gpurun_out/mode.json 2> gpurun_out/mode.err
    python -c "
import json; d=json.loads(open('gpurun_out/mode.json').read().strip().splitlines()[-1])
print('$C', '[$M]', 'ms', round(d['ms_per_step'],2), 'pairs/s %.3e' % d['value'], 'dtw_eval_frac', round(d['prune']['dtw_evaluated_frac'],5), 'dtw_ms', round(d['stage_ms']['ms_dtw'],2), 'cells', d['walk']['dtw_cells_computed'])" 2>&1 | tail -1
  done
done
