#!/bin/bash
# Late round-2 evidence on the final build: GPU suite, smoke, bench line,
# reference arm, launch list of a short bench run.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; echo "rc=$?" >> gpurun_out/smoke.txt
timeout 900 python bench.py > gpurun_out/bench.txt 2>&1; echo "rc=$?" >> gpurun_out/bench.txt
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.txt 2>&1; echo "rc=$?" >> gpurun_out/bench_ref.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-configs --no-traffic > gpurun_out/launches.log 2>&1
tail -2 gpurun_out/pytest_gpu.txt; tail -2 gpurun_out/smoke.txt; tail -c 400 gpurun_out/bench.txt; tail -c 300 gpurun_out/bench_ref.txt
