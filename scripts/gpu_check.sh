#!/bin/bash
# GPU tests + C5 bench with and without the pre-filter (plain runs, no profiler).
python -m pytest tests -m gpu -x -q ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_gpu.log
python bench.py --no-cpu-baseline --steps 2 --warmup 3 > gpurun_out/bench_pf.json 2> gpurun_out/bench_pf.err; echo "bench rc=$?"; cat gpurun_out/bench_pf.json; tail -3 gpurun_out/bench_pf.err
python bench.py --no-cpu-baseline --steps 2 --warmup 3 --no-prefilter > gpurun_out/bench_nopf.json 2> gpurun_out/bench_nopf.err; echo "bench nopf rc=$?"; cat gpurun_out/bench_nopf.json; tail -3 gpurun_out/bench_nopf.err
