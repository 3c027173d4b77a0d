# clip bench (cache vs no cache) + full GPU tests
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/clip
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/clip/tests.log 2>&1; echo tests=$?
for c in ${CFGS:-cfg4 cfg5}; do
  timeout 300 python bench.py --config $c --clip-frames 8 --steps 5 --warmup 3 > gpurun_out/clip/clip_$c.log 2>&1
  timeout 300 python bench.py --config $c --clip-frames 8 --no-cache --steps 5 --warmup 3 > gpurun_out/clip/clipnc_$c.log 2>&1
done
tail -n 2 gpurun_out/clip/tests.log
for f in gpurun_out/clip/clip*.log; do python - "$f" <<'PY'
import json, sys
for l in open(sys.argv[1]):
    if l.startswith('{'):
        d = json.loads(l); print(sys.argv[1], round(d['ms_per_step'], 2), round(d['frames_per_s'], 1), d.get('gpu_launches'))
PY
done
