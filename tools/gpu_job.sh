mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_ops_gpu.py -x -q > gpurun_out/pytest_ops.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_ops.txt
