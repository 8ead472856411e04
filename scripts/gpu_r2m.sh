#!/bin/bash
timeout 1800 python -m pytest tests/test_gpu_search.py tests/test_gpu_shards.py tests/test_gpu_kernels.py -x -q > gpurun_out/r2m_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r2m_tests.log
for C in C5 C3 C4; do
timeout 900 python bench.py --config $C --no-cpu-baseline > gpurun_out/r2m_$C.json 2> gpurun_out/r2m_$C.err; echo "$C rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/r2m_$C.json').read().strip().splitlines()[-1])
print('ms', d['ms_per_step'], 'steps', d['step_ms']); print({k: round(v,2) for k,v in d['stage_ms'].items()})"
done
timeout 600 python bench.py --config C3 --w 100 --no-cpu-baseline > gpurun_out/r2m_C3w100.json 2> gpurun_out/r2m_C3w100.err; echo "C3w100 rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/r2m_C3w100.json').read().strip().splitlines()[-1])
print('ms', d['ms_per_step']); print({k: round(v,2) for k,v in d['stage_ms'].items()}); print(d['walk'], d['prune'])"
timeout 1200 python scripts/shard_projection.py --config C5 --gpus 2,4,8 > gpurun_out/r2m_shard_projection.json 2> gpurun_out/r2m_shard_projection.err; echo "projection rc=$?"; tail -4 gpurun_out/r2m_shard_projection.err
