#!/bin/bash
# round-2 evidence: GPU suite, scalar-call latency, bench (with the in-run
# traffic probe), the launch list of a short bench
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q --durations=15 > gpurun_out/pytest_gpu.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.txt
timeout 300 python tools/scalar_latency.py > gpurun_out/scalar.txt 2>&1
timeout 1200 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.txt 2>&1; echo "rc=$?" >> gpurun_out/bench.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-configs --no-operators --no-traffic --no-e2e > gpurun_out/launch_bench.txt 2>&1
