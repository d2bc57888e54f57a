mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_observability_gpu.py tests/test_ops_gpu.py -q > gpurun_out/pytest_all.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_all.txt
