#!/bin/bash
# engine-parallel kernel: golden-case parity first, then the smoke entry point
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -40 > gpurun_out/parity.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1
