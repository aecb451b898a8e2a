cd $GRAFT_REPO_ROOT
for v in "" "HPAC_HOOK_NO_STREAM=1"; do
env $v BENCH_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29655 bench.py --gpus 2 --workload kmeans --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline 2>/dev/null | grep -o '"quality": {[^}]*}\|"iterations": {[^}]*}'
done
timeout 600 python bench.py --workload kmeans --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline 2>/dev/null | grep -o '"quality": {[^}]*}\|"iterations": {[^}]*}'
