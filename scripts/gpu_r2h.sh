#!/bin/bash
timeout 120 ./scripts/isa_probe > gpurun_out/r2h_isa_probe.txt 2>&1; echo "isa rc=$?"; grep "gate\|DTW\|LB" gpurun_out/r2h_isa_probe.txt
DTWLB_DEBUG_SPANS=1 timeout 900 python bench.py --no-cpu-baseline > gpurun_out/r2h_C5.json 2> gpurun_out/r2h_C5.err; echo "C5 rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/r2h_C5.json').read().strip().splitlines()[-1])
print('ms', d['ms_per_step'], 'steps', d['step_ms']); print({k: round(v,2) for k,v in d['stage_ms'].items()})"
grep "setup->first\|query block" gpurun_out/r2h_C5.err | sort | uniq -c | sort -rn | head
timeout 1200 python scripts/shard_projection.py --config C5 --gpus 2,4,8 > gpurun_out/r2h_shard_projection.json 2> gpurun_out/r2h_shard_projection.err; echo "projection rc=$?"; cat gpurun_out/r2h_shard_projection.err | tail -4
