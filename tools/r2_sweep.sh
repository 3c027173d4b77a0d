# frames in flight x K2 residency cap sweep of the resident bench step (cfg2)
cd $GRAFT_REPO_ROOT
for f in 2 3 4; do for c in 0 2 3 4; do
  TS_FRAMES_IN_FLIGHT=$f TS_K2_CTAS_PER_SM=$c timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu --no-e2e > gpurun_out/r2_sweep_f${f}_c${c}.json 2>/dev/null
done; done
