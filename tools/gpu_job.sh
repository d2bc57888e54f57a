mkdir -p gpurun_out
rm -f gpurun_out/occ.txt
for k in 2 3 4 2 3 4; do
  echo "== ctas/sm $k" >> gpurun_out/occ.txt
  NX_SIM_CTAS_PER_SM=$k timeout 300 python bench.py --no-cpu-baseline --no-e2e --no-operators >> gpurun_out/occ.txt 2>&1
done
