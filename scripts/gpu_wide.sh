#!/bin/bash
# Wide-band DTW + stream kernel (R rows per lane): parity, App. B timing, C3 at w = 100, C5-stream.
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -k "wide or dtw_band" > gpurun_out/pytest_wide.log 2>&1; echo "pytest wide rc=$?"; tail -3 gpurun_out/pytest_wide.log
timeout 600 python -m pytest tests/test_gpu_search.py -x -q -k "wide" > gpurun_out/pytest_wide2.log 2>&1; echo "pytest walk rc=$?"; tail -3 gpurun_out/pytest_wide2.log
timeout 600 python -m pytest tests/test_gpu_stream.py tests/test_gpu_appendix_b.py -x -q > gpurun_out/pytest_wide3.log 2>&1; echo "pytest stream/appB rc=$?"; tail -3 gpurun_out/pytest_wide3.log
timeout 300 python scripts/appendix_b.py 100000 --no-oracle > gpurun_out/appendix_b.json 2>&1; echo "appB rc=$?"; cat gpurun_out/appendix_b.json | python -c "import json,sys; d=json.load(sys.stdin); print({k:(round(v['violation_frac'],4), '%.3g cells/s' % v['cells_per_s'], round(v['seconds']*1e3,2)) for k,v in d.items()})"
timeout 300 python bench.py --config C3 --w 100 --no-cpu-baseline --steps 3 --warmup 3 > gpurun_out/b_C3w100.json 2>&1; echo "C3w100 rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/b_C3w100.json').read().strip().splitlines()[-1]); r=d['roofline']
print('C3w100 ms', round(d['ms_per_step'],1), {k:(round(r[k]['ms'],2), round(r[k]['frac'],3)) for k in ('bound_pass','survivor_kernel','dtw_kernel') if k in r}, d['walk'])"
for q in 1 2 4 8; do
  timeout 300 python bench.py --config C5s$q --no-cpu-baseline --steps 10 --warmup 3 --db-index > gpurun_out/b4_C5s${q}_idx.json 2>&1; echo "C5s$q idx rc=$?"
done
python - <<'PY'
import json, glob
for f in sorted(glob.glob('gpurun_out/b4_*.json')):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, 'ERR', e); continue
    r = d['roofline']
    print(f, 'ms %.3f' % d['ms_per_step'], 'bound %.3f ms frac %.3f' % (r['bound_pass']['ms'], r['bound_pass']['frac']),
          'dom', r['dominant'], {k: round(v, 3) for k, v in d['stage_ms'].items()}, 'rounds', d['walk']['walk_rounds'])
PY
