mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest_gpu.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.txt
timeout 900 python bench.py --no-cpu-baseline --no-e2e --no-operators > gpurun_out/bench_1.txt 2>&1
timeout 900 python bench.py --no-cpu-baseline --no-e2e --no-operators > gpurun_out/bench_2.txt 2>&1
timeout 300 python tools/timeline.py --replicas 512 > gpurun_out/tl512.txt 2>&1
