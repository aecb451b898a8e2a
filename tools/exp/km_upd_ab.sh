# A/B of K-Means update-kernel variants (tools/variants/<name>) on the C3 Lloyd loop
for v in default $VARIANTS; do
  if [ $v = default ]; then L=; else L=tools/variants/$v/libhpac_b200.so; fi
  echo "== $v"; env ${L:+HPAC_LIB=$L} timeout 600 python tools/exp/run_lloyd_c3.py 2>&1 | tail -2
done
