#!/bin/bash
timeout 1800 python -m pytest tests/test_gpu_shards.py tests/test_gpu_search.py -x -q > gpurun_out/r2l_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r2l_tests.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/r2l_C5.json 2> gpurun_out/r2l_C5.err; echo "C5 rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/r2l_C5.json').read().strip().splitlines()[-1])
print('ms', d['ms_per_step'], 'steps', d['step_ms']); print({k: round(v,2) for k,v in d['stage_ms'].items()})"
timeout 1200 python scripts/shard_projection.py --config C5 --gpus 2,4,8 > gpurun_out/r2l_shard_projection.json 2> gpurun_out/r2l_shard_projection.err; echo "projection rc=$?"; tail -4 gpurun_out/r2l_shard_projection.err
