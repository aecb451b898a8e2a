O=gpurun_out; mkdir -p $O; T=${TAG:-r02j}
for ts in 2 8; do
 SPEC=iact TSIZE=$ts timeout 300 ncu --set full --import-source on --clock-control none -k regex:bs_iact -s 1 -c 1 -o $O/${T}_iact_t$ts -f python tools/exp/bs_one.py > /dev/null 2>&1
 ncu -i $O/${T}_iact_t$ts.ncu-rep --page details --csv > $O/${T}_iact_t${ts}_details.csv
 ncu -i $O/${T}_iact_t$ts.ncu-rep --page raw --csv > $O/${T}_iact_t${ts}_raw.csv
 ncu -i $O/${T}_iact_t$ts.ncu-rep --page source --csv --print-source sass > $O/${T}_iact_t${ts}_source.csv
 rm -f $O/${T}_iact_t$ts.ncu-rep
done
