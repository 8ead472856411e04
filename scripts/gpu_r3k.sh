#!/bin/bash
# 8-GPU projection from one-GPU shard timings with this session's kernels
timeout 2400 python scripts/shard_projection.py --config C5 --gpus 2,4,8 > gpurun_out/r3k_shard_projection.json 2> gpurun_out/r3k_shard_projection.err; echo "proj rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/r3k_shard_projection.json'))
print('one_gpu_ms', d['one_gpu_ms'])
for p in d['projections']: print(p['gpus'], 'max shard %.1f' % p['max_shard_ms'], 'proj %.1f' % p['projected_step_ms'], 'x%.2f' % p['projected_speedup'], 'bitid', p['sharded_result_bit_identical'], 'qshard x%.2f' % p['query_sharded']['projected_speedup'])" || tail -5 gpurun_out/r3k_shard_projection.err
