#!/bin/bash
# Stall comparison: lockstep kernel at 1 replica/SM vs the full 512 shard.
mkdir -p gpurun_out
for n in 148 512; do
  timeout 900 ncu --section WarpStateStats --section SchedulerStats --section InstructionStats \
    --section MemoryWorkloadAnalysis --section MemoryWorkloadAnalysis_Tables --section SourceCounters --section LaunchStats --section Occupancy \
    --clock-control none --import-source on -k nx_sim_kernel -c 1 -o gpurun_out/sim_n$n \
    python tools/prof_sim.py --replicas $n --requests 2000 > gpurun_out/ncu_n$n.log 2>&1
done
