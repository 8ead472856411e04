#!/bin/bash
# after the 8x walk growth default: GPU suite, smoke, bench lines, shard projection
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/r3u_gpu_tests.log 2>&1; echo "gpu tests rc=$?"; tail -2 gpurun_out/r3u_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r3u_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r3u_smoke.log
timeout 900 python bench.py > gpurun_out/r3u_C5_bench.json 2> gpurun_out/r3u_C5_bench.err; echo "C5 rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/r3u_C5_bench.json').read().strip().splitlines()[-1])
print('C5 ms %.2f value %.4g e2e %.4g frac %.3f' % (d['ms_per_step'], d['value'], d['e2e']['value'], d['roofline']['frac']), d['step_ms'], d['clocks'])"
for cw in "C4 51" "C3 50" "C3 100" "C5s1 25" "C5s8 25" "C2p1 25" "C2p2 25"; do
set -- $cw
timeout 600 python bench.py --config $1 --w $2 --no-cpu-baseline > gpurun_out/r3u_$1_w$2.json 2> gpurun_out/r3u_$1_w$2.err
python -c "
import json; d=json.loads(open('gpurun_out/r3u_$1_w$2.json').read().strip().splitlines()[-1])
print('$1 w=$2 ms %.3f' % d['ms_per_step'], 'dtw_kernel %.2f' % d['stage_ms']['ms_dtw_kernel'], d['roofline']['kernel'][:30], 'frac %.3f' % d['roofline']['frac'])"
done
timeout 1200 python scripts/shard_projection.py --config C5 --gpus 2,4,8 > gpurun_out/r3u_shard_projection.json 2> gpurun_out/r3u_shard_projection.err; echo "proj rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/r3u_shard_projection.json'))
print('one_gpu_ms', d['one_gpu_ms'])
for p in d['projections']: print(p['gpus'], 'max shard %.1f' % p['max_shard_ms'], 'proj %.1f' % p['projected_step_ms'], 'x%.2f' % p['projected_speedup'], 'bitid', p['sharded_result_bit_identical'], 'qshard x%.2f' % p['query_sharded']['projected_speedup'])"
