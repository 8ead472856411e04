#!/bin/bash
# fp16-staged survivor pass (128-candidate tiles): parity, then C5 / C2p2 with DTWLB_SURV_H16 = 1, 0
timeout 1200 python -m pytest tests/test_gpu_search.py tests/test_gpu_kernels.py tests/test_gpu_shards.py tests/test_gpu_stream.py -x -q > gpurun_out/r3a_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r3a_tests.log
for cfg in C5 C2p2; do
for h in 1 0; do
DTWLB_SURV_H16=$h timeout 600 python bench.py --config $cfg --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/r3a_${cfg}_h$h.json 2> gpurun_out/r3a_${cfg}_h$h.err
python -c "
import json; d=json.loads(open('gpurun_out/r3a_${cfg}_h$h.json').read().strip().splitlines()[-1])
print('$cfg h16=$h ms %.1f' % d['ms_per_step'], {k: round(v,1) for k,v in d['stage_ms'].items()}, 'impr %.4f dtw %.5f' % (d['prune']['improved_evaluated_frac'], d['prune']['dtw_evaluated_frac']))" || tail -5 gpurun_out/r3a_${cfg}_h$h.err
done; done
