# A/B on one box: alternate the default library and $ALT (relative to the package dir)
mkdir -p gpurun_out; : > gpurun_out/ab.txt
for i in 1 2 3; do
  for v in new base; do
    if [ $v = base ]; then export NX_SO=$ALT; else unset NX_SO; fi
    timeout 600 python bench.py --no-cpu-baseline --no-e2e --no-operators 2>/dev/null | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['value'])" >> gpurun_out/ab.txt
  done
done
