# ncu --set full of the Blackscholes C1 lane kernel (exact) and the iACT lane kernel
O=gpurun_out; mkdir -p $O; T=${TAG:-r04a}
for spec in exact iact; do
  k=$([ $spec = exact ] && echo "regex:bs_lane_kernel" || echo "regex:bs_iact_lane")
  SPEC=$spec timeout 300 ncu --set full --import-source on --clock-control none -k $k -s 1 -c 1 -o $O/${T}_bs_$spec -f python tools/exp/bs_one.py > /dev/null 2>&1
  ncu -i $O/${T}_bs_$spec.ncu-rep --page details --csv > $O/${T}_bs_${spec}_details.csv
  ncu -i $O/${T}_bs_$spec.ncu-rep --page raw --csv > $O/${T}_bs_${spec}_raw.csv
  ncu -i $O/${T}_bs_$spec.ncu-rep --page source --csv --print-source sass > $O/${T}_bs_${spec}_source.csv
done
