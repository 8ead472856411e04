#!/bin/bash
# fused survivor pass A/B: parity tests, then C5 / C4 / C3 with DTWLB_SURV_FUSED = 0, 1, 2
timeout 900 python -m pytest tests/test_gpu_search.py tests/test_gpu_kernels.py tests/test_gpu_shards.py -x -q > gpurun_out/r2v_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r2v_tests.log
for cfg in C5 C4 C3; do
for f in 0 1 2; do
DTWLB_SURV_FUSED=$f timeout 600 python bench.py --config $cfg --no-cpu-baseline --steps 3 --warmup 3 > gpurun_out/r2v_${cfg}_f$f.json 2> gpurun_out/r2v_${cfg}_f$f.err
python -c "
import json; d=json.loads(open('gpurun_out/r2v_${cfg}_f$f.json').read().strip().splitlines()[-1])
print('$cfg fused=$f ms %.1f' % d['ms_per_step'], {k: round(v,1) for k,v in d['stage_ms'].items()}, 'dtw_eval', d['walk']['dtw_evaluated'])"
done; done
