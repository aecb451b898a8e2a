#!/bin/bash
# One GPU session: bench lines + ncu launch list + one full capture of the
# dominant kernel of every workload. Usage (under gpurun):
#   bash tools/profile_round.sh TAG            (then: python tools/profile_post.py TAG)
TAG=${1:-r01}
O=gpurun_out
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > $O/${TAG}_gpu.txt 2>&1
B="python bench.py"
Q="--e2e-steps 0 --no-cpu-baseline"
# ---- bench lines (timed, not under a profiler); SKIP_BENCH=1 skips them
if [ -z "$SKIP_BENCH" ]; then
timeout 900 $B --steps 5 --warmup 3 > $O/${TAG}_bench_binomial.json 2> $O/${TAG}_bench_binomial.err
timeout 600 $B --workload blackscholes --steps 10 --warmup 5 > $O/${TAG}_bench_blackscholes.json 2> $O/${TAG}_bench_blackscholes.err
timeout 600 $B --workload lavamd --steps 3 --warmup 2 > $O/${TAG}_bench_lavamd.json 2> $O/${TAG}_bench_lavamd.err
timeout 900 $B --workload kmeans --steps 2 --warmup 1 > $O/${TAG}_bench_kmeans.json 2> $O/${TAG}_bench_kmeans.err
timeout 600 $B --workload kmeans-region --steps 5 --warmup 3 > $O/${TAG}_bench_kmeans-region.json 2> $O/${TAG}_bench_kmeans-region.err
fi
# ---- launch list of the default bench command (cold-cache, serialised: compare shares)
[ -z "$CAPS" ] && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/${TAG}_launches_binomial.csv \
  $B --steps 2 --warmup 1 $Q > /dev/null 2>&1
# ---- one full capture of each workload's timed kernel
cap() {  # name, kernel regex, skip, bench args...   (CAPS=regex: only matching names)
  local name=$1 rx=$2 skip=$3; shift 3
  if [ -n "$CAPS" ] && ! [[ $name =~ $CAPS ]]; then return; fi
  timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
    -k "regex:$rx" -s $skip -c 1 -o $O/${TAG}_$name -f $B "$@" $Q > $O/${TAG}_$name.log 2>&1
  ncu -i $O/${TAG}_$name.ncu-rep --page raw --csv > $O/${TAG}_${name}_raw.csv 2>/dev/null
  ncu -i $O/${TAG}_$name.ncu-rep --page details --csv > $O/${TAG}_${name}_details.csv 2>/dev/null
  ncu -i $O/${TAG}_$name.ncu-rep --page source --csv --print-source sass > $O/${TAG}_${name}_source.csv 2>/dev/null
  rm -f $O/${TAG}_$name.ncu-rep
}
# approximate kernels: the exact arm runs first (warmup+steps launches of the
# TECH=3 kernel), so the first matching launch of the approximate kernel is
# the warm-up of the timed arm
# binomial (non-TAF): decide -> price -> resolve; the lattice kernel is the
# price kernel (exact arm first: warmup+steps launches, then the iACT arm)
cap binomial_iact 'binomial_price_kernel' 2 --steps 1 --warmup 1
cap binomial_exact 'binomial_price_kernel' 0 --steps 1 --warmup 1
cap bs_taf 'bs_lane_kernel<.int.0' 0 --workload blackscholes --steps 1 --warmup 1
cap bs_exact 'bs_lane_kernel<.int.3' 0 --workload blackscholes --steps 1 --warmup 1
cap lavamd_taf 'engine_thread_kernel<hpac::AppLavaMD, .int.0' 0 --workload lavamd --steps 1 --warmup 1
cap lavamd_exact 'engine_thread_kernel<hpac::AppLavaMD, .int.3' 0 --workload lavamd --steps 1 --warmup 1
# the Lloyd loop runs as a CUDA graph with a conditional node, whose kernel
# nodes ncu cannot profile: capture the host-driven loop (same kernels)
export HPAC_KMEANS_HOST_LOOP=1
cap kmeans_region 'engine_thread_kernel<hpac::AppKmeansDmma, .int.2' 3 --workload kmeans --steps 1 --warmup 1
cap kmeans_update 'kmeans_update_partial' 3 --workload kmeans --steps 1 --warmup 1
cap kmeans_compact 'kmeans_changed_compact' 3 --workload kmeans --steps 1 --warmup 1
unset HPAC_KMEANS_HOST_LOOP
ls -la $O
