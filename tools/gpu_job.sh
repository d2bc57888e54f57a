mkdir -p gpurun_out
rm -f gpurun_out/excl.txt
for k in 48 64 24 48 64 32; do
  echo "== excl $k" >> gpurun_out/excl.txt
  NX_EXCL_SMS=$k timeout 300 python bench.py --no-cpu-baseline --no-e2e --no-operators >> gpurun_out/excl.txt 2>&1
done
