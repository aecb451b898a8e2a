# A/B of Blackscholes lane-kernel variants (tools/variants/<name>) on C1
for v in default $VARIANTS; do
  if [ $v = default ]; then L=; else L=tools/variants/$v/libhpac_b200.so; fi
  echo "== $v"; env ${L:+HPAC_LIB=$L} HPAC_STREAM_TMA=0 timeout 300 python tools/exp/run_bs_lane.py 0 2>&1 | grep -v iact
done
