#!/bin/bash
# round-2 (late): GPU suite, smoke, bench line, K1 ncu capture
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; echo "rc=$?" >> gpurun_out/smoke.txt
timeout 900 python bench.py > gpurun_out/bench.txt 2>&1; echo "rc=$?" >> gpurun_out/bench.txt
timeout 600 ncu --set full --import-source on --clock-control none -k regex:perf_eval_kernel -s 4 -c 1 \
  -o gpurun_out/k1 -f python tools/k1_check.py > gpurun_out/k1prof.txt 2>&1
ncu -i gpurun_out/k1.ncu-rep --page raw --csv > gpurun_out/k1_raw.csv 2>/dev/null
tail -3 gpurun_out/pytest_gpu.txt; tail -2 gpurun_out/smoke.txt; tail -c 600 gpurun_out/bench.txt
