#!/bin/bash
# full GPU suite, then a short bench of the engine-parallel kernel
mkdir -p gpurun_out
export NX_DEBUG=1
timeout 1500 python -m pytest tests -m gpu -q -x --durations=10 > gpurun_out/pytest_gpu.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.txt
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-operators > gpurun_out/bench.txt 2>&1; echo "rc=$?" >> gpurun_out/bench.txt
