mkdir -p gpurun_out
timeout 300 python tools/k1_check.py > gpurun_out/k1.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "perf or k1 or eval" > gpurun_out/pytest_k1.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_k1.txt
