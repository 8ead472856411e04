#!/bin/bash
# ISA pipe rates; C5 with the top-k merge early exit; stream variants; multi-GPU projection.
timeout 120 ./scripts/isa_probe > gpurun_out/r2e_isa_probe.txt 2>&1; echo "isa rc=$?"; cat gpurun_out/r2e_isa_probe.txt
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/r2e_C5.json 2> gpurun_out/r2e_C5.err; echo "C5 rc=$?"
for v in 1 3; do for D in 0 3 4; do
  DTWLB_STREAM_SQ=$v DTWLB_STREAM_STAGES=$D timeout 300 python bench.py --config C5s8 --no-cpu-baseline --steps 10 --warmup 3 --db-index > gpurun_out/r2e_C5s8_sq${v}_D$D.json 2>&1; echo "C5s8 sq$v D$D rc=$?"
done; done
DTWLB_STREAM_SQ=2 timeout 300 python bench.py --config C5s4 --no-cpu-baseline --steps 10 --warmup 3 --db-index > gpurun_out/r2e_C5s4_sq2.json 2>&1; echo "C5s4 sq2 rc=$?"
timeout 300 python bench.py --config C5s4 --no-cpu-baseline --steps 10 --warmup 3 --db-index > gpurun_out/r2e_C5s4.json 2>&1; echo "C5s4 rc=$?"
python - <<'PY'
import json, glob
for f in sorted(glob.glob('gpurun_out/r2e_C*.json')):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, 'ERR', e); continue
    r = d['roofline']; b = r.get('bound_pass', {})
    print(f, 'ms %.3f' % d['ms_per_step'], 'bound %.3f ms frac %.3f' % (b.get('ms', 0), b.get('frac', 0)),
          {k: round(v, 2) for k, v in d['stage_ms'].items()})
PY
timeout 1200 python scripts/shard_projection.py --config C5 --gpus 2,4,8 > gpurun_out/r2e_shard_projection.json 2> gpurun_out/r2e_shard_projection.err; echo "projection rc=$?"; tail -30 gpurun_out/r2e_shard_projection.json
