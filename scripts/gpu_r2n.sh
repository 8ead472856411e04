#!/bin/bash
for S in 256 512 1024; do
  for C in C3 C4 C5; do
    DTWLB_SEED=$S timeout 600 python bench.py --config $C --no-cpu-baseline --steps 5 > gpurun_out/r2n_${C}_S$S.json 2>/dev/null
    python -c "
import json; d=json.loads(open('gpurun_out/r2n_${C}_S$S.json').read().strip().splitlines()[-1])
print('$C S=$S ms', round(d['ms_per_step'],2), {k: round(v,2) for k,v in d['stage_ms'].items() if k in ('ms_improved','ms_dtw','ms_dtw_kernel')})"
  done
  DTWLB_SEED=$S timeout 600 python bench.py --config C3 --w 100 --no-cpu-baseline --steps 5 > gpurun_out/r2n_C3w100_S$S.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/r2n_C3w100_S$S.json').read().strip().splitlines()[-1])
print('C3w100 S=$S ms', round(d['ms_per_step'],2), {k: round(v,2) for k,v in d['stage_ms'].items() if k in ('ms_improved','ms_dtw','ms_dtw_kernel')}, d['walk']['range1_dtw'], d['walk']['dtw_evaluated'])"
done
timeout 1200 python scripts/shard_projection.py --config C5 --gpus 4,8 > gpurun_out/r2n_shard_projection.json 2> gpurun_out/r2n_shard_projection.err; echo "projection rc=$?"; tail -3 gpurun_out/r2n_shard_projection.err
python -c "
import json; d=json.load(open('gpurun_out/r2n_shard_projection.json'))
for p in d['projections']: print(p['gpus'], p['shard_rep_ms'])"
