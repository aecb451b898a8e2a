for v in default $VARIANTS; do
  if [ $v = default ]; then L=; else L=tools/variants/$v/libhpac_b200.so; fi
  echo "== $v"; env ${L:+HPAC_LIB=$L} timeout 600 python tools/exp/run_bino_taf.py 2>&1 | tail -2
done
