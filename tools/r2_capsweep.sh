# K2 residency cap x frames in flight sweep per config (resident step only)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/cap
for c in ${CFGS:-cfg5 cfg4 cfg3}; do
  for fl in 2 3; do for cap in 0 2 3 4 5; do
    TS_FRAMES_IN_FLIGHT=$fl TS_K2_CTAS_PER_SM=$cap timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c fl=$fl cap=$cap', round(d['ms_per_step'],3))"
  done; done
done
