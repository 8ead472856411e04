#!/bin/bash
# survivor kernel: fixed-point REDUX group sums (DTWLB_SURV_FX = 1 vs 0)
timeout 1200 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_search.py tests/test_gpu_shards.py tests/test_gpu_stream.py -x -q > gpurun_out/r3q_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r3q_tests.log
for cfg in C5 C4 C3; do
for f in 1 0; do
DTWLB_SURV_FX=$f timeout 600 python bench.py --config $cfg --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/r3q_${cfg}_fx$f.json 2> gpurun_out/r3q_${cfg}_fx$f.err
python -c "
import json; d=json.loads(open('gpurun_out/r3q_${cfg}_fx$f.json').read().strip().splitlines()[-1])
print('$cfg fx=$f ms %.1f' % d['ms_per_step'], 'surv %.2f' % d['stage_ms']['ms_survivor_kernel'], 'impr %.5f dtw %.5f cells %.4g' % (d['prune']['improved_evaluated_frac'], d['prune']['dtw_evaluated_frac'], d['walk']['dtw_cells_computed']))"
done; done
