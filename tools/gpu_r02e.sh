#!/bin/bash
# round-2 diagnostics on the final build: phase/window/refit attribution and
# an ncu --set full capture of nx_sim_kernel (one wave of 148 replicas) + K1
mkdir -p gpurun_out
timeout 300 python tools/pdes_report.py --shard 512 > gpurun_out/pdes.txt 2>&1
timeout 300 python tools/merge_probe.py > gpurun_out/mp.txt 2>&1
timeout 300 python tools/refit_probe.py > gpurun_out/rp.txt 2>&1
bash tools/gpu_prof_pdes.sh
bash tools/gpu_prof_k1.sh
ncu -i gpurun_out/sim_pdes.ncu-rep --page details --csv > gpurun_out/sim_pdes_details.csv 2>/dev/null
