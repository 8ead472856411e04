#!/bin/bash
timeout 1200 python -m pytest tests/test_gpu_search.py tests/test_gpu_kernels.py -x -q -k "host or wide or eight or oracle_cache" > gpurun_out/r2p_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r2p_tests.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/r2p_C5.json 2> gpurun_out/r2p_C5.err; echo "C5 rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/r2p_C5.json').read().strip().splitlines()[-1])
print('ms', d['ms_per_step'], 'value %.4g' % d['value'], 'e2e %.4g' % d['e2e']['value'], 'e2e ms %.2f' % (8192e6/d['e2e']['value']*1e3))"
CMD="python bench.py --config C3 --w 100 --steps 1 --warmup 2 --no-cpu-baseline"
R=gpurun_out/r2p_C3w100_wide
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dtw_wide -s 10 -c 1 -o $R $CMD > gpurun_out/r2p_ncu_wide.log 2>&1; echo "ncu wide rc=$?"
python scripts/ncu_summary.py $R.ncu-rep > ${R}_ncu.txt 2>&1; python scripts/ncu_lines.py $R.ncu-rep 30 > ${R}_lines.txt 2>&1
R=gpurun_out/r2p_appb_wide
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dtw_wide -s 2 -c 1 -o $R python scripts/appendix_b.py 100000 --no-oracle > gpurun_out/r2p_ncu_appb.log 2>&1; echo "ncu appb rc=$?"
python scripts/ncu_summary.py $R.ncu-rep > ${R}_ncu.txt 2>&1; python scripts/ncu_lines.py $R.ncu-rep 30 > ${R}_lines.txt 2>&1
head -30 gpurun_out/r2p_C3w100_wide_ncu.txt; head -30 gpurun_out/r2p_appb_wide_ncu.txt
