#!/bin/bash
# end-of-round check of the committed tree: GPU suite, smoke, default bench line
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/r3p_gpu_tests.log 2>&1; echo "gpu tests rc=$?"; tail -2 gpurun_out/r3p_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r3p_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r3p_smoke.log
timeout 900 python bench.py > gpurun_out/r3p_C5_bench.json 2> gpurun_out/r3p_C5_bench.err; echo "C5 rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/r3p_C5_bench.json').read().strip().splitlines()[-1])
print('C5 ms %.2f value %.4g e2e %.4g frac %.3f mix %.3f' % (d['ms_per_step'], d['value'], d['e2e']['value'], d['roofline']['frac'], d['roofline']['frac_of_mix_peak']), d['step_ms'], d['clocks'], d['achieved_fraction']['fraction_at_mix_peak'], d['cpu_baseline']['value'])"
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r3p_ref.json 2> gpurun_out/r3p_ref.err; echo "ref rc=$?"; tail -1 gpurun_out/r3p_ref.json | cut -c1-300
