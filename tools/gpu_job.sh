mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; echo "rc=$?" >> gpurun_out/smoke.txt
timeout 900 python bench.py > gpurun_out/bench.txt 2>&1; echo "rc=$?" >> gpurun_out/bench.txt
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.txt 2>&1; echo "rc=$?" >> gpurun_out/bench_ref.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-operators > gpurun_out/launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:perf_eval_kernel -c 1 -o gpurun_out/k1_final python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-operators > gpurun_out/ncu_k1.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k nx_sim_kernel -c 1 -o gpurun_out/sim_final python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-operators > gpurun_out/ncu_sim.log 2>&1
