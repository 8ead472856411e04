#!/bin/bash
timeout 900 python bench.py > gpurun_out/r2i_C5.json 2> gpurun_out/r2i_C5.err; echo "C5 rc=$?"
for C in C5s1 C5s8 C3 C4; do
  timeout 600 python bench.py --config $C --no-cpu-baseline > gpurun_out/r2i_$C.json 2> gpurun_out/r2i_$C.err; echo "$C rc=$?"
done
python - <<'PY'
import json, glob
for f in sorted(glob.glob('gpurun_out/r2i_C*.json')):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, 'ERR', e); continue
    r = d['roofline']
    print(f, 'ms %.3f' % d['ms_per_step'], 'dom', r['dominant'], round(r['frac'], 3), r.get('frac_of_mix_peak'),
          {k: (round(r[k]['ms'], 2), round(r[k]['frac'], 3), round(r[k].get('frac_of_mix_peak', 0), 3)) for k in r if isinstance(r[k], dict) and 'ms' in r[k]})
    print('   steps', d['step_ms'])
PY
timeout 1200 python scripts/shard_projection.py --config C5 --gpus 2,4,8 > gpurun_out/r2i_shard_projection.json 2> gpurun_out/r2i_shard_projection.err; echo "projection rc=$?"; cat gpurun_out/r2i_shard_projection.err | tail -4
