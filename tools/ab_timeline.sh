#!/bin/bash
# A/B of two library builds: per-replica timelines at several shard sizes.
mkdir -p gpurun_out
for so in _nxsched.so _nxsched_inl.so; do
  for n in 512 148 32; do
    echo "== $so n=$n" >> gpurun_out/ab.txt
    NX_SO=$so timeout 300 python tools/timeline.py --replicas $n >> gpurun_out/ab.txt 2>&1
  done
done
