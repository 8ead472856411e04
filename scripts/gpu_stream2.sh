#!/bin/bash
# C5-stream round 2: correctness of the TMA-box stream kernel + envelope rewrite, then bench lines
# for the three copy engines, then ncu of the stream kernel and the envelope kernel.
python -m pytest tests/test_gpu_stream.py tests/test_gpu_kernels.py -x -q > gpurun_out/pytest_stream2.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_stream2.log
for q in 1 8; do
  for c in 2 1 0; do
    DTWLB_STREAM_COPY=$c python bench.py --config C5s$q --no-cpu-baseline --steps 5 --warmup 3 --db-index > gpurun_out/b2_C5s${q}_c$c.json 2>&1; echo "C5s$q copy$c rc=$?"
  done
done
python bench.py --config C5s8 --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/b2_C5s8_noidx.json 2>&1; echo "noidx rc=$?"
python - <<'PY'
import json, glob
for f in sorted(glob.glob('gpurun_out/b2_*.json')):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, 'ERR', e); continue
    r = d['roofline']
    print(f, 'ms %.3f' % d['ms_per_step'], 'bound %.3f ms frac %.3f' % (r['bound_pass']['ms'], r['bound_pass']['frac']),
          'dom', r['dominant'], {k: round(v, 3) for k, v in d['stage_ms'].items()}, 'rounds', d['walk']['walk_rounds'])
PY
python bench.py --config C5s8 --steps 1 --warmup 1 --no-cpu-baseline --db-index > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:keogh_stream -c 2 -o gpurun_out/stream_tma python bench.py --config C5s8 --steps 1 --warmup 1 --no-cpu-baseline --db-index > gpurun_out/ncu_stream.log 2>&1; echo "ncu rc=$?"
