#!/bin/bash
# w sweep with this round's kernels
for cw in "C5 13" "C5 51" "C4 26" "C4 51" "C3 25" "C3 50"; do
set -- $cw
timeout 900 python bench.py --config $1 --w $2 --no-cpu-baseline --steps 3 --warmup 3 > gpurun_out/r3o_$1_w$2.json 2> gpurun_out/r3o_$1_w$2.err
python -c "
import json; d=json.loads(open('gpurun_out/r3o_$1_w$2.json').read().strip().splitlines()[-1])
print('$1 w=$2 ms %.1f pairs/s %.3g dtw_eval %.4f dtw_kernel %.1f gate %.1f surv %.1f' % (d['ms_per_step'], d['value'], d['prune']['dtw_evaluated_frac']*100, d['stage_ms']['ms_dtw_kernel'], d['stage_ms']['ms_keogh'], d['stage_ms']['ms_survivor_kernel']))" || tail -3 gpurun_out/r3o_$1_w$2.err
done
