#!/bin/bash
mkdir -p gpurun_out
export NX_DEBUG=1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1
