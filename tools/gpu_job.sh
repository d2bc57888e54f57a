mkdir -p gpurun_out
NX_SO=_nxsched_fx.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_ops_gpu.py tests/test_observability_gpu.py -q > gpurun_out/pytest_fx.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_fx.txt
NX_SO=_nxsched_fx.so timeout 900 python bench.py --no-cpu-baseline --no-e2e --no-operators > gpurun_out/bench_fx1.txt 2>&1
timeout 900 python bench.py --no-cpu-baseline --no-e2e --no-operators > gpurun_out/bench_base.txt 2>&1
NX_SO=_nxsched_fx.so timeout 900 python bench.py --no-cpu-baseline --no-e2e --no-operators > gpurun_out/bench_fx2.txt 2>&1
NX_SO=_nxsched_fx.so timeout 300 python tools/phase_report.py > gpurun_out/phase_fx.txt 2>&1
