mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_k6_gpu.py -q > gpurun_out/pytest_k6.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_k6.txt
