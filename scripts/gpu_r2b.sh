#!/bin/bash
# Round-2 checkpoint: full GPU suite, smoke, bench lines (C5 default, C5-stream, C3/C4, C3 w=100, Appendix B),
# launch list of the default C5 bench, ncu --set full of the dominant kernels.
T="timeout 1500"
$T python -m pytest tests -m gpu -x -q > gpurun_out/r2b_gpu_tests.log 2>&1; echo "gpu tests rc=$?"; tail -3 gpurun_out/r2b_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2b_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/r2b_C5.json 2> gpurun_out/r2b_C5.err; echo "C5 rc=$?"
for C in C5s1 C5s2 C5s4 C5s8; do
  timeout 300 python bench.py --config $C --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/r2b_$C.json 2> gpurun_out/r2b_$C.err; echo "$C rc=$?"
done
for C in C3 C4 C2p1 C2p2; do
  timeout 600 python bench.py --config $C --no-cpu-baseline > gpurun_out/r2b_$C.json 2> gpurun_out/r2b_$C.err; echo "$C rc=$?"
done
timeout 600 python bench.py --config C3 --w 100 --no-cpu-baseline --steps 3 --warmup 3 > gpurun_out/r2b_C3w100.json 2> gpurun_out/r2b_C3w100.err; echo "C3w100 rc=$?"
timeout 300 python scripts/appendix_b.py 100000 --no-oracle > gpurun_out/r2b_appendix_b.json 2>&1; echo "appB rc=$?"
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2b_C5_launches.csv $CMD > gpurun_out/r2b_ncu_launch.log 2>&1; echo "launch list rc=$?"
for KS in improved_kernel:7 dtw4_kernel:40 keogh_tile_kernel:3; do
  K=${KS%%:*}; S=${KS##*:}
  R=gpurun_out/r2b_C5_${K}_$S
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s $S -c 1 -o $R $CMD > gpurun_out/r2b_ncu_${K}.log 2>&1
  echo "full $K rc=$?"
  python scripts/ncu_summary.py $R.ncu-rep > ${R}_ncu.txt 2>&1
  python scripts/ncu_lines.py $R.ncu-rep 40 > ${R}_lines.txt 2>&1
done
CMD="python bench.py --config C5s1 --steps 1 --warmup 3 --no-cpu-baseline"
R=gpurun_out/r2b_C5s1_stream
timeout 600 ncu --set full --clock-control none --import-source on -k regex:stream -s 3 -c 1 -o $R $CMD > gpurun_out/r2b_ncu_stream.log 2>&1; echo "full stream rc=$?"
python scripts/ncu_summary.py $R.ncu-rep > ${R}_ncu.txt 2>&1
