#!/bin/bash
# GPU tests + C5 bench (pre-filter default) + launch list of a 1-step run.
python -m pytest tests -m gpu -x -q ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
python bench.py --no-cpu-baseline --steps 2 --warmup 3 ${BENCH_ARGS} > gpurun_out/bench_q.json 2> gpurun_out/bench_q.err; echo "bench rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/bench_q.json').read().strip().splitlines()[-1])
print('ms', round(d['ms_per_step'],1), {k: round(v,1) for k,v in d['stage_ms'].items()}, 'cells', d['walk']['dtw_cells_computed'], 'dtw_eval', d['walk']['dtw_evaluated'])"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/q_launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline ${BENCH_ARGS} > /dev/null 2>&1; echo "launch rc=$?"
python scripts/launch_summary.py gpurun_out/q_launches.csv 4 | head -10
