#!/bin/bash
# first walk batch per query (DTWLB_D0) sweep
for cfg in C5 C4 C3; do
for d in 16 32 64 128; do
DTWLB_D0=$d timeout 600 python bench.py --config $cfg --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/r3f_${cfg}_d$d.json 2> gpurun_out/r3f_${cfg}_d$d.err
python -c "
import json; d=json.loads(open('gpurun_out/r3f_${cfg}_d$d.json').read().strip().splitlines()[-1])
print('$cfg d0=$d ms %.1f' % d['ms_per_step'], 'dtw %.1f kern %.1f' % (d['stage_ms']['ms_dtw'], d['stage_ms']['ms_dtw_kernel']), 'cells %.4g r1cells %.4g rounds %d' % (d['walk']['dtw_cells_computed'], d['walk']['range1_cells'], d['walk']['walk_rounds']))"
done; done
