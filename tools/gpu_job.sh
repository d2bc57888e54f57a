mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_ops_gpu.py tests/test_observability_gpu.py -q > gpurun_out/pytest_gpu.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.txt
timeout 300 python tools/phase_report.py > gpurun_out/phase.txt 2>&1
timeout 900 python bench.py --no-cpu-baseline --no-e2e --no-operators > gpurun_out/bench_1.txt 2>&1
