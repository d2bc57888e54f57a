mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench.txt 2>&1; echo "rc=$?" >> gpurun_out/bench.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:perf_eval_kernel -c 1 -o gpurun_out/k1_r01b python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/ncu_k1.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k nx_sim_kernel -c 1 -o gpurun_out/sim_r01b python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/ncu_sim.log 2>&1
