#!/bin/bash
# first walk batch (DTWLB_D0) for C3 at w = 100 (wide kernel, ~2e5 cells per pair, k = 1)
for d in 4 8 16 32 128; do
DTWLB_D0=$d timeout 600 python bench.py --config C3 --w 100 --no-cpu-baseline --steps 3 --warmup 3 > gpurun_out/r3r_d$d.json 2> gpurun_out/r3r_d$d.err
python -c "
import json; d=json.loads(open('gpurun_out/r3r_d$d.json').read().strip().splitlines()[-1])
print('C3w100 d0=$d ms %.1f dtw_kernel %.1f cells %.4g r1cells %.4g rounds %d' % (d['ms_per_step'], d['stage_ms']['ms_dtw_kernel'], d['walk']['dtw_cells_computed'], d['walk']['range1_cells'], d['walk']['walk_rounds']))"
done
