#!/bin/bash
# Round-2 checkpoint: wide DTW (fixed), fused gate, p=4, stream; benches; dtw4 range-2 ncu.
T="timeout 900"
$T python -m pytest tests/test_gpu_kernels.py -x -q > gpurun_out/r2a_kernels.log 2>&1; echo "kernels rc=$?"; tail -2 gpurun_out/r2a_kernels.log
$T python -m pytest tests/test_gpu_search.py tests/test_gpu_shards.py tests/test_gpu_stream.py tests/test_gpu_appendix_b.py -x -q > gpurun_out/r2a_search.log 2>&1; echo "search rc=$?"; tail -2 gpurun_out/r2a_search.log
timeout 300 python scripts/appendix_b.py 100000 --no-oracle > gpurun_out/appendix_b.json 2>&1; echo "appB rc=$?"; python -c "import json; d=json.load(open('gpurun_out/appendix_b.json')); print({k:(round(v['violation_frac'],4), '%.3g cells/s' % v['cells_per_s'], round(v['seconds']*1e3,2)) for k,v in d.items()})"
timeout 600 python bench.py --config C3 --w 100 --no-cpu-baseline --steps 3 --warmup 3 > gpurun_out/r2a_C3w100.json 2>&1; echo "C3w100 rc=$?"
timeout 600 python bench.py --no-cpu-baseline --steps 3 --warmup 3 > gpurun_out/r2a_C5.json 2>&1; echo "C5 rc=$?"
timeout 300 python bench.py --config C5s4 --no-cpu-baseline --steps 10 --warmup 3 --db-index > gpurun_out/r2a_C5s4.json 2>&1; echo "C5s4 rc=$?"
timeout 300 python bench.py --config C5s8 --no-cpu-baseline --steps 10 --warmup 3 --db-index > gpurun_out/r2a_C5s8.json 2>&1; echo "C5s8 rc=$?"
python - <<'PY'
import json, glob
for f in sorted(glob.glob('gpurun_out/r2a_*.json')):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, 'ERR', e); continue
    r = d['roofline']
    print(f, 'ms %.3f' % d['ms_per_step'], 'dom', r['dominant'],
          {k: (round(r[k]['ms'], 3), round(r[k]['frac'], 3)) for k in ('bound_pass', 'survivor_kernel', 'dtw_kernel') if k in r},
          {k: round(v, 2) for k, v in d['stage_ms'].items()})
PY
timeout 600 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dtw4 -s 13 -c 1 -o gpurun_out/r2a_dtw4_r2 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/r2a_ncu.log 2>&1; echo "ncu rc=$?"
