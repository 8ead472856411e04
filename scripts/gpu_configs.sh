#!/bin/bash
# tests, then one bench line per config (plain runs).
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
for C in ${CONFIGS:-C5 C3 C4 C2p1 C2p2 C1}; do
  python bench.py --config $C --no-cpu-baseline --steps ${STEPS:-3} --warmup 3 ${BENCH_ARGS} > gpurun_out/cfg_$C.json 2> gpurun_out/cfg_$C.err
  echo "$C rc=$?"
  python -c "
import json; d=json.loads(open('gpurun_out/cfg_$C.json').read().strip().splitlines()[-1])
print('$C', 'ms', round(d['ms_per_step'],2), 'value %.3e' % d['value'], 'e2e %.3e' % d['e2e']['value'], {k: round(v,2) for k,v in d['stage_ms'].items()}, 'frac', round(d['roofline']['frac'],3), d['prune'])" 2>&1 | tail -1
done
