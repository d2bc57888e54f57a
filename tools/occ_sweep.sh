#!/bin/bash
# Occupancy sweep of the lockstep kernel (diagnostic): bench at capped CTAs/SM.
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.txt
timeout 300 python tools/phase_report.py > gpurun_out/phase.txt 2>&1
for k in ${OCC_LIST:-2 3 4 6}; do
  echo "== ctas/sm $k" >> gpurun_out/occ.txt
  NX_SIM_CTAS_PER_SM=$k timeout 300 python bench.py --no-cpu-baseline --no-e2e >> gpurun_out/occ.txt 2>&1
done
