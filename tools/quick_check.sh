mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_observability_gpu.py tests/test_ops_gpu.py -x -q > gpurun_out/pytest_q.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_q.txt
for i in 1 2; do timeout 600 python bench.py --no-cpu-baseline --no-e2e --no-operators > gpurun_out/bench_q$i.txt 2>&1; done
timeout 300 python tools/phase_report.py > gpurun_out/phase_q.txt 2>&1
