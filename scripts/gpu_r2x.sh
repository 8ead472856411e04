#!/bin/bash
# midpoint-form gate: parity (kernels, search, stream, shards), then C5 / C4 / C3 / C2 bench lines
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2x_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r2x_tests.log
for cfg in C5 C4 C3 C2p2; do
timeout 600 python bench.py --config $cfg --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/r2x_${cfg}.json 2> gpurun_out/r2x_${cfg}.err
python -c "
import json; d=json.loads(open('gpurun_out/r2x_${cfg}.json').read().strip().splitlines()[-1])
print('$cfg ms %.1f' % d['ms_per_step'], {k: round(v,1) for k,v in d['stage_ms'].items()}, 'gate frac %.3f mix %.3f' % (d['roofline']['bound_pass']['frac'], d['roofline']['bound_pass'].get('frac_of_mix_peak', 0)), 'keogh_eval %.4f' % d['prune']['keogh_evaluated_frac'])"
done
./scripts/isa_probe > gpurun_out/r2x_isa_probe.txt 2>&1; tail -3 gpurun_out/r2x_isa_probe.txt
