# A/B of LavaMD variants (tools/variants/<name>) at B1^3 boxes (default 48)
for v in default $VARIANTS; do
  if [ $v = default ]; then L=; else L=tools/variants/$v/libhpac_b200.so; fi
  echo "== $v"; env ${L:+HPAC_LIB=$L} B1=${B1:-48} REPS=3 timeout 600 python tools/exp/run_lava.py 2>&1 | tail -2
done
