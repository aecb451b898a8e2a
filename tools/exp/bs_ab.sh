for v in default $VARIANTS default; do
  if [ $v = default ]; then L=; else L=tools/variants/$v/libhpac_b200.so; fi
  echo "== $v"; env ${L:+HPAC_LIB=$L} timeout 300 python tools/exp/run_bs_pair.py 0 2>&1 | grep -E "exact|taf\(" 
  env ${L:+HPAC_LIB=$L} HPAC_ENGINE=auto timeout 300 python tools/exp/run_bs_iact3.py auto 2>&1 | grep -E "iact\(2,0.5,thread"
done
