#!/bin/bash
# C5-stream (Q <= 8) checks: GPU tests touching the bound passes, bench lines for Q in {1,2,4,8}
# (with / without the prebuilt database index, TMA bulk vs cp.async copies), a C5 regression
# line, and the launch list of a C5s8 step.
python -m pytest tests/test_gpu_stream.py tests/test_gpu_kernels.py tests/test_gpu_search.py -x -q > gpurun_out/pytest_stream.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_stream.log
for q in 1 2 4 8; do
  python bench.py --config C5s$q --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/b_C5s$q.json 2> gpurun_out/b_C5s$q.err; echo "C5s$q rc=$?"
  python bench.py --config C5s$q --no-cpu-baseline --steps 5 --warmup 3 --db-index > gpurun_out/b_C5s${q}_idx.json 2> gpurun_out/b_C5s${q}_idx.err; echo "C5s$q idx rc=$?"
done
DTWLB_STREAM_COPY=1 python bench.py --config C5s8 --no-cpu-baseline --steps 5 --warmup 3 --db-index > gpurun_out/b_C5s8_cpasync.json 2>&1; echo "cpasync rc=$?"
python bench.py --config C5s8 --no-cpu-baseline --steps 5 --warmup 3 --db-index --no-stream > gpurun_out/b_C5s8_nostream.json 2>&1; echo "nostream rc=$?"
python - <<'PY'
import json, glob
for f in sorted(glob.glob('gpurun_out/b_C5s*.json')):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, 'ERR', e); continue
    r = d['roofline']
    print(f, 'ms %.3f' % d['ms_per_step'], 'bound %.3f ms frac %.3f' % (r['bound_pass']['ms'], r['bound_pass']['frac']),
          'dom', r['dominant'], {k: round(v, 3) for k, v in d['stage_ms'].items()})
PY
python bench.py --no-cpu-baseline --steps 2 --warmup 3 > gpurun_out/b_C5.json 2> gpurun_out/b_C5.err; echo "C5 rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/b_C5.json').read().strip().splitlines()[-1]); r=d['roofline']
print('C5 ms', round(d['ms_per_step'],1), 'dom', r['dominant'], {k:(round(r[k]['ms'],1), round(r[k]['frac'],3)) for k in ('bound_pass','survivor_kernel','dtw_kernel')})"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/C5s8_launches.csv python bench.py --config C5s8 --steps 1 --warmup 1 --no-cpu-baseline --db-index > /dev/null 2>&1; echo "launch rc=$?"
python scripts/launch_summary.py gpurun_out/C5s8_launches.csv 2 | head -20
