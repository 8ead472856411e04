#!/bin/bash
timeout 120 ./scripts/isa_probe > gpurun_out/r2f_isa_probe.txt 2>&1; echo "isa rc=$?"; cat gpurun_out/r2f_isa_probe.txt
DTWLB_DEBUG_SPANS=1 timeout 900 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/r2f_C5.json 2> gpurun_out/r2f_C5.err; echo "C5 rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/r2f_C5.json').read().strip().splitlines()[-1])
print('ms', d['ms_per_step'], 'steps', d['step_ms']); print({k: round(v,2) for k,v in d['stage_ms'].items()})"
grep -c "events" gpurun_out/r2f_C5.err; grep "events" gpurun_out/r2f_C5.err | awk '{ if ($6+0 > 2.0) print }' | head -40
timeout 900 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/r2f_C5_plain.json 2> gpurun_out/r2f_C5_plain.err; echo "C5 plain rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/r2f_C5_plain.json').read().strip().splitlines()[-1])
print('ms', d['ms_per_step'], 'steps', d['step_ms']); print({k: round(v,2) for k,v in d['stage_ms'].items()})"
DTWLB_BENCH_NO_CLOCKS=1 timeout 900 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/r2f_C5_noclk.json 2> gpurun_out/r2f_C5_noclk.err; echo "C5 noclk rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/r2f_C5_noclk.json').read().strip().splitlines()[-1])
print('ms', d['ms_per_step'], 'steps', d['step_ms']); print({k: round(v,2) for k,v in d['stage_ms'].items()})"
