#!/bin/bash
# Stream kernels after the LDS fix + the split-query shared-box kernel (Q = 5..8).
timeout 900 python -m pytest tests/test_gpu_stream.py -x -q > gpurun_out/r2d_stream_tests.log 2>&1; echo "stream tests rc=$?"; tail -2 gpurun_out/r2d_stream_tests.log
for C in C5s1 C5s2 C5s4 C5s8; do
  timeout 300 python bench.py --config $C --no-cpu-baseline --steps 10 --warmup 3 --db-index > gpurun_out/r2d_$C.json 2> gpurun_out/r2d_$C.err; echo "$C rc=$?"
done
for C in C5s4 C5s8; do
  DTWLB_STREAM_SQ=0 timeout 300 python bench.py --config $C --no-cpu-baseline --steps 10 --warmup 3 --db-index > gpurun_out/r2d_${C}_sq0.json 2>&1; echo "$C sq0 rc=$?"
  DTWLB_STREAM_SQ=2 timeout 300 python bench.py --config $C --no-cpu-baseline --steps 10 --warmup 3 --db-index > gpurun_out/r2d_${C}_sq2.json 2>&1; echo "$C sq2 rc=$?"
done
python - <<'PY'
import json, glob
for f in sorted(glob.glob('gpurun_out/r2d_C*.json')):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, 'ERR', e); continue
    r = d['roofline']; b = r.get('bound_pass', {})
    print(f, 'ms %.3f' % d['ms_per_step'], 'bound %.3f ms frac %.3f' % (b.get('ms', 0), b.get('frac', 0)),
          {k: round(v, 3) for k, v in d['stage_ms'].items()})
PY
CMD="python bench.py --config C5s8 --steps 1 --warmup 3 --no-cpu-baseline --db-index"
R=gpurun_out/r2d_C5s8_stream
timeout 600 ncu --set full --clock-control none --import-source on -k regex:stream -s 3 -c 1 -o $R $CMD > gpurun_out/r2d_ncu_stream.log 2>&1; echo "full stream rc=$?"
python scripts/ncu_summary.py $R.ncu-rep > ${R}_ncu.txt 2>&1
