# frames in flight x K2 residency cap sweep of the resident bench step
cd $GRAFT_REPO_ROOT
for c in ${CFG:-cfg2}; do
for f in 2 3 4; do for k in 0 3; do
  TS_FRAMES_IN_FLIGHT=$f TS_K2_CTAS_PER_SM=$k timeout 300 python bench.py --config $c --steps 30 --warmup 5 --no-cpu --no-e2e > gpurun_out/r2_sweep_${c}_f${f}_c${k}.json 2>/dev/null
done; done
done
