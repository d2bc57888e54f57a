for v in "" 4 5 6; do
  if [ -z "$v" ]; then so=""; else so="NX_SO=$PWD/tools/_var$v/_nxsched.so"; fi
  echo "ctas ${v:-3}: $(env $so timeout 120 python tools/k1_check.py 2>&1 | grep '^K1')"
done
