#!/bin/bash
run() { # cfg w d0 gs
  DTWLB_D0=$3 DTWLB_WALK_GS=$4 timeout 600 python bench.py --config $1 --w $2 --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/r3t_$1_w$2_d$3_g$4.json 2> gpurun_out/r3t_$1_w$2_d$3_g$4.err
  python -c "
import json; d=json.loads(open('gpurun_out/r3t_$1_w$2_d$3_g$4.json').read().strip().splitlines()[-1])
print('$1 w=$2 d0=$3 gs=$4 ms %.1f dtw_kernel %.1f dtw %.1f cells %.4g rounds %d' % (d['ms_per_step'], d['stage_ms']['ms_dtw_kernel'], d['stage_ms']['ms_dtw'], d['walk']['dtw_cells_computed'], d['walk']['walk_rounds']))"
}
run C5 25 128 2; run C5 25 128 3; run C4 51 128 3; run C3 100 128 4; run C5 51 128 1; run C5 51 128 2; run C5 51 128 3; run C4 26 128 1; run C4 26 128 3
