#!/bin/bash
# final tree: the other configs, the 8-GPU projection, ncu --set full of the largest DTW walk launch
for cw in "C4 51" "C4 26" "C3 50" "C3 25" "C3 100" "C5 13" "C5 51" "C5s1 25" "C5s2 25" "C5s4 25" "C5s8 25" "C2p1 25" "C2p2 25"; do
set -- $cw
timeout 600 python bench.py --config $1 --w $2 --no-cpu-baseline > gpurun_out/r02zi_$1_w$2.json 2> gpurun_out/r02zi_$1_w$2.err
python -c "
import json; d=json.loads(open('gpurun_out/r02zi_$1_w$2.json').read().strip().splitlines()[-1])
s=d['stage_ms']; print('$1 w=$2 ms %.3f' % d['ms_per_step'], 'gate %.2f surv %.2f dtw_kernel %.2f' % (s['ms_keogh'], s['ms_survivor_kernel'], s['ms_dtw_kernel']), d['roofline']['kernel'][:30], 'frac %.3f' % d['roofline']['frac'])" 2>&1 | tail -1
done
timeout 1200 python scripts/shard_projection.py --config C5 --gpus 2,4,8 > gpurun_out/r02zi_shard_projection.json 2> gpurun_out/r02zi_shard_projection.err; echo "proj rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/r02zi_shard_projection.json'))
print('one_gpu_ms', d['one_gpu_ms'])
for p in d['projections']: print(p['gpus'], 'max shard %.1f' % p['max_shard_ms'], 'proj %.1f' % p['projected_step_ms'], 'x%.2f' % p['projected_speedup'], 'bitid', p['sharded_result_bit_identical'], 'qshard x%.2f' % p['query_sharded']['projected_speedup'])"
timeout 300 python scripts/appendix_b.py > gpurun_out/r02zi_appendix_b.json 2> gpurun_out/r02zi_appendix_b.err; echo "appB rc=$?"; tail -c 400 gpurun_out/r02zi_appendix_b.json
CMD="python bench.py --config C5 --steps 1 --warmup 3 --no-cpu-baseline"
K=dtw4_kernel; S=10; R=gpurun_out/r02zi_C5_${K}_$S
ncu --set full --clock-control none --import-source on -k regex:$K -s $S -c 1 -o $R $CMD > gpurun_out/r02zi_ncu_${K}_$S.log 2>&1
echo "full $K skip $S rc=$?"
python scripts/ncu_summary.py $R.ncu-rep > ${R}_ncu.txt 2>&1
python scripts/ncu_lines.py $R.ncu-rep 40 > ${R}_lines.txt 2>&1
ncu -i $R.ncu-rep --page raw --csv > ${R}_raw.csv 2>/dev/null
rm -f $R.ncu-rep
