#!/bin/bash
# end-of-round check of the final tree + its launch list and survivor-kernel capture
bash scripts/gpu_r3p.sh
for f in gpu_tests.log smoke.log C5_bench.json C5_bench.err ref.json ref.err; do mv gpurun_out/r3p_$f gpurun_out/r02zk_$f; done
TAG=r02zk CFG=C5 CAPTURES="improved_kernel:1" bash scripts/profile_round.sh > gpurun_out/r02zk_profile.log 2>&1; tail -3 gpurun_out/r02zk_profile.log
python scripts/launch_summary.py gpurun_out/r02zk_C5_launches.csv 6 > gpurun_out/r02zk_C5_launch_summary.txt 2>&1; head -6 gpurun_out/r02zk_C5_launch_summary.txt
timeout 1200 python scripts/shard_projection.py --config C5 --gpus 8 > gpurun_out/r02zk_shard_projection.json 2> gpurun_out/r02zk_shard_projection.err; echo "proj rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/r02zk_shard_projection.json'))
print('one_gpu_ms', d['one_gpu_ms'])
for p in d['projections']: print(p['gpus'], 'max shard %.1f' % p['max_shard_ms'], 'proj %.1f' % p['projected_step_ms'], 'x%.2f' % p['projected_speedup'], 'bitid', p['sharded_result_bit_identical'], 'qshard x%.2f' % p['query_sharded']['projected_speedup'])"
