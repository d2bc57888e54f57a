#!/bin/bash
mkdir -p gpurun_out
for n in 1 148; do
  timeout 600 ncu --set full --clock-control none -k nx_sim_kernel -c 1 -o gpurun_out/load$n -f python tools/load_ncu_child.py $n > gpurun_out/load_ncu$n.txt 2>&1
  ncu -i gpurun_out/load$n.ncu-rep --page raw --csv > gpurun_out/load${n}_raw.csv 2>/dev/null
done
