#!/bin/bash
# K1 A/B: the in-tree build vs variant .so files (tools/_var*), alternating,
# plus the K1 parity tests and one ncu --set full capture of the in-tree kernel.
mkdir -p gpurun_out
{
for i in 1 2 3; do
  echo "new: $(timeout 120 python tools/k1_check.py 2>&1 | grep '^K1')"
  for v in ${K1_VARS:-old}; do
    echo "$v: $(NX_SO=$PWD/tools/_var$v/_nxsched.so timeout 120 python tools/k1_check.py 2>&1 | grep '^K1')"
  done
done
timeout 120 python tools/k1_check.py 2>&1 | grep -v '^K1'
timeout 300 python -m pytest -q -x tests/test_gpu_parity.py -k k1 2>&1 | tail -3
} > gpurun_out/k1ab.txt 2>&1
if [ -z "$NO_NCU" ]; then
timeout 600 ncu --set full --import-source on --clock-control none -k regex:perf_eval_kernel -s 4 -c 1 \
  -o gpurun_out/k1 -f python tools/k1_check.py > gpurun_out/k1prof.txt 2>&1
ncu -i gpurun_out/k1.ncu-rep --page raw --csv > gpurun_out/k1_raw.csv 2>/dev/null
fi
cat gpurun_out/k1ab.txt
