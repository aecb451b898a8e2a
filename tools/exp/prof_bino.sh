# ncu capture of the binomial iACT kernel for one library variant: VAR=name TAG=tag
O=gpurun_out; mkdir -p $O; T=${TAG:-r02s}
L=; [ -n "$VAR" ] && L=tools/variants/$VAR/libhpac_b200.so
env ${L:+HPAC_LIB=$L} timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
  -k 'regex:binomial_team_kernel<.int.1' -s 0 -c 1 -o $O/${T}_bino_${VAR:-default} -f python bench.py --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline --sub-configs off > $O/${T}_bino_${VAR:-default}.log 2>&1
ncu -i $O/${T}_bino_${VAR:-default}.ncu-rep --page raw --csv > $O/${T}_bino_${VAR:-default}_raw.csv
ncu -i $O/${T}_bino_${VAR:-default}.ncu-rep --page details --csv > $O/${T}_bino_${VAR:-default}_details.csv
ncu -i $O/${T}_bino_${VAR:-default}.ncu-rep --page source --csv --print-source sass > $O/${T}_bino_${VAR:-default}_source.csv
rm -f $O/${T}_bino_${VAR:-default}.ncu-rep
