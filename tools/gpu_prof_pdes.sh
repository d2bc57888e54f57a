#!/bin/bash
# ncu stall profile of the engine-parallel simulation kernel on 148 replicas (one wave)
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k nx_sim_kernel -c 1 \
  -o gpurun_out/sim_pdes -f python tools/prof_sim.py --replicas ${PROF_REPLICAS:-148} --requests ${PROF_REQUESTS:-1000} > gpurun_out/prof.txt 2>&1
ncu -i gpurun_out/sim_pdes.ncu-rep --page source --print-source cuda,sass --csv > gpurun_out/sim_pdes_source.csv 2>/dev/null
ncu -i gpurun_out/sim_pdes.ncu-rep --page raw --csv > gpurun_out/sim_pdes_raw.csv 2>/dev/null
rm -f gpurun_out/sim_pdes_source.csv.gz; gzip -f gpurun_out/sim_pdes_source.csv
