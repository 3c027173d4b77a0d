# A/B of the K3 split on the bench's updates-only path (TS_K3_SPLIT=1 forced vs the automatic choice)
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
for c in ${CFGS:-cfg2 cfg3}; do
for r in 1 2; do
timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-e2e --no-cpu > gpurun_out/k3ab_auto_${c}_$r.json 2>/dev/null
TS_K3_SPLIT=1 timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-e2e --no-cpu > gpurun_out/k3ab_split_${c}_$r.json 2>/dev/null
done
done
