#!/bin/bash
# DTW prefetch (PF) A/B + fused survivor pass: full GPU suite, then C5 / C4 / C3 with DTWLB_DTW_PF = 0, 1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2w_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r2w_tests.log
for cfg in C5 C4 C3; do
for f in 0 1; do
DTWLB_DTW_PF=$f timeout 600 python bench.py --config $cfg --no-cpu-baseline --steps 3 --warmup 3 > gpurun_out/r2w_${cfg}_pf$f.json 2> gpurun_out/r2w_${cfg}_pf$f.err
python -c "
import json; d=json.loads(open('gpurun_out/r2w_${cfg}_pf$f.json').read().strip().splitlines()[-1])
print('$cfg pf=$f ms %.1f' % d['ms_per_step'], {k: round(v,1) for k,v in d['stage_ms'].items()}, 'cells %.4g' % d['walk']['dtw_cells_computed'], 'frac %.3f' % d['roofline']['frac'])"
done; done
