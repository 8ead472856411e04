#!/bin/bash
# final-tree profile (launch list + ncu --set full of the survivor and DTW kernels) and a
# re-sweep of the range plan with the column abandon schedule (seed size, ranges, walk growth)
TAG=r02zi CFG=C5 CAPTURES="improved_kernel:1 dtw4_kernel:13" bash scripts/profile_round.sh
python scripts/launch_summary.py gpurun_out/r02zi_C5_launches.csv 5 > gpurun_out/r02zi_C5_launch_summary.txt 2>&1
run() {  # label, env assignments...
  local label=$1; shift
  env "$@" timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r3v_$label.json 2> gpurun_out/r3v_$label.err
  python -c "
import json; d=json.loads(open('gpurun_out/r3v_$label.json').read().strip().splitlines()[-1])
s=d['stage_ms']; print('$label ms %.2f' % d['ms_per_step'], 'gate %.1f sel %.1f surv %.1f dtwk %.1f' % (s['ms_keogh'], s['ms_select'], s['ms_survivor_kernel'], s['ms_dtw_kernel']), 'rounds', d['walk']['walk_rounds'])" 2>&1 | tail -1
}
run base DTWLB_NOP=1
for S in 512 900 2048 3072; do run seed$S DTWLB_SEED=$S; done
run ranges3 DTWLB_RANGES=3
run ranges3g16 DTWLB_RANGES=3 DTWLB_RANGE_GROWTH=16
for G in 4 16; do run gs$G DTWLB_WALK_GS=$G; done
for D in 32 128; do run d0_$D DTWLB_D0=$D; done
