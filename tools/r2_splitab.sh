# K3 single pass vs split (touched list + compact fits read by K4) per config
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/splitab
for c in ${CFGS:-cfg2 cfg3 cfg4}; do
  for sp in 0 1; do
    TS_K3_SPLIT=$sp timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu --no-e2e > gpurun_out/splitab/${c}_$sp.json 2> gpurun_out/splitab/${c}_$sp.err
  done
done
for f in gpurun_out/splitab/*.json; do python - "$f" <<'PY'
import json, sys
for l in open(sys.argv[1]):
    if l.startswith('{'):
        d = json.loads(l); print(sys.argv[1], round(d['ms_per_step'], 3), d.get('frame_latency_ms'), d.get('stage_ms'))
PY
done
