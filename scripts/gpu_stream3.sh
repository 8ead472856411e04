#!/bin/bash
# C5-stream round 3: swizzled-TMA stream kernel; Q = 1, 2, 4, 8 with the prebuilt index and without.
python -m pytest tests/test_gpu_stream.py -x -q > gpurun_out/pytest_stream3.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_stream3.log
for q in 1 2 4 8; do
  python bench.py --config C5s$q --no-cpu-baseline --steps 10 --warmup 3 --db-index > gpurun_out/b3_C5s${q}_idx.json 2>&1; echo "C5s$q idx rc=$?"
  python bench.py --config C5s$q --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/b3_C5s${q}.json 2>&1; echo "C5s$q rc=$?"
done
python - <<'PY'
import json, glob
for f in sorted(glob.glob('gpurun_out/b3_*.json')):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, 'ERR', e); continue
    r = d['roofline']
    print(f, 'ms %.3f' % d['ms_per_step'], 'bound %.3f ms frac %.3f' % (r['bound_pass']['ms'], r['bound_pass']['frac']),
          'dom', r['dominant'], {k: round(v, 3) for k, v in d['stage_ms'].items()}, 'rounds', d['walk']['walk_rounds'], 'e2e', round(d['e2e']['value']/1e9,2))
PY
python bench.py --config C5s4 --steps 1 --warmup 1 --no-cpu-baseline --db-index > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:keogh_stream -c 1 -o gpurun_out/stream_swz4 python bench.py --config C5s4 --steps 1 --warmup 1 --no-cpu-baseline --db-index > gpurun_out/ncu_stream3.log 2>&1; echo "ncu rc=$?"
