# ncu --set full of the LavaMD exact and TAF-warp launches (B1^3 boxes, default 32)
O=gpurun_out; mkdir -p $O; T=${TAG:-r04c}
B1=${B1:-32} timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k regex:AppLavaMD -c 2 -o $O/${T}_lava -f python tools/exp/run_lava.py > /dev/null 2>&1
ncu -i $O/${T}_lava.ncu-rep --page raw --csv > $O/${T}_lava_raw.csv
ncu -i $O/${T}_lava.ncu-rep --page details --csv > $O/${T}_lava_details.csv
ncu -i $O/${T}_lava.ncu-rep --page source --csv --print-source sass > $O/${T}_lava_source.csv
