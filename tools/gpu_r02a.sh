#!/bin/bash
# round-2 check: full GPU suite, then the bench (N=1) and its reference arm
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
nproc > gpurun_out/nproc.txt; lscpu | head -20 >> gpurun_out/nproc.txt
timeout 1500 python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/pytest_gpu.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.txt
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.txt 2>&1; echo "rc=$?" >> gpurun_out/bench.txt
