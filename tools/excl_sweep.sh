mkdir -p gpurun_out; : > gpurun_out/excl.txt
for i in 1 2; do for e in 32 24 16 40; do
  NX_EXCL_SMS=$e timeout 600 python bench.py --no-cpu-baseline --no-e2e --no-operators 2>/dev/null | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$e', d['value'])" >> gpurun_out/excl.txt
done; done
timeout 300 python tools/phase_report.py > gpurun_out/phase.txt 2>&1
