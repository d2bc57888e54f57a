#!/bin/bash
# ncu of the K1 evaluator at 2^26 records (k1_check's timed launches)
mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:perf_eval_kernel -s 4 -c 1 \
  -o gpurun_out/k1 -f python tools/k1_check.py > gpurun_out/k1prof.txt 2>&1
ncu -i gpurun_out/k1.ncu-rep --page raw --csv > gpurun_out/k1_raw.csv 2>/dev/null
ncu -i gpurun_out/k1.ncu-rep --page details --csv > gpurun_out/k1_details.csv 2>/dev/null
