#!/bin/bash
# One GPU session: bench lines + ncu launch list + one full capture per hot kernel.
# Usage (under gpurun): bash tools/profile_round.sh TAG
TAG=${1:-r01}
O=gpurun_out
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > $O/${TAG}_gpu.txt 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 > $O/${TAG}_bench_binomial.json 2> $O/${TAG}_bench_binomial.err
timeout 600 python bench.py --workload blackscholes --steps 10 --warmup 5 > $O/${TAG}_bench_bs.json 2> $O/${TAG}_bench_bs.err
timeout 900 python bench.py --workload kmeans --steps 5 --warmup 3 > $O/${TAG}_bench_km.json 2> $O/${TAG}_bench_km.err
# launch list of the bench command (cold-cache, serialised: compare shares)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/${TAG}_launches_binomial.csv \
  python bench.py --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1
# full captures (one launch each): exact lattice and the iACT region
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
  -k 'regex:binomial_team_kernel<3' -c 1 -o $O/${TAG}_bino_exact -f \
  python bench.py --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
  -k 'regex:binomial_team_kernel<1' -c 1 -o $O/${TAG}_bino_iact -f \
  python bench.py --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
  -k 'regex:engine_thread_kernel' -s 2 -c 1 -o $O/${TAG}_bs_taf -f \
  python bench.py --workload blackscholes --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
  -k 'regex:engine_thread_kernel' -s 2 -c 1 -o $O/${TAG}_km_region -f \
  python bench.py --workload kmeans --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1
# reduce reports to CSV pages (the box returns <= 64 MiB); keep only the iACT rep
for r in $O/${TAG}_*.ncu-rep; do
  b=${r%.ncu-rep}
  ncu -i $r --page raw --csv > ${b}_raw.csv 2>/dev/null
  ncu -i $r --page details --csv > ${b}_details.csv 2>/dev/null
  ncu -i $r --page source --csv --print-source sass > ${b}_source.csv 2>/dev/null
  case $r in *bino_iact*) ;; *) rm -f $r ;; esac
done
gzip -f $O/${TAG}_*_source.csv
ls -la $O
