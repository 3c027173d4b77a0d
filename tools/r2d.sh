cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2d
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/r2d/tests.log 2>&1; echo tests=$?
tail -2 gpurun_out/r2d/tests.log
timeout 600 python bench.py --config cfg5 --steps 10 --warmup 3 --no-cpu > gpurun_out/r2d/cfg5.json 2> gpurun_out/r2d/cfg5.err
timeout 600 python bench.py --config cfg5 --clip-frames 8 --steps 3 --warmup 3 > gpurun_out/r2d/cfg5_clip.json 2> gpurun_out/r2d/cfg5_clip.err
timeout 600 python bench.py --config cfg4 --clip-frames 8 --steps 5 --warmup 3 > gpurun_out/r2d/cfg4_clip.json 2> gpurun_out/r2d/cfg4_clip.err
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/r2d/cfg2.json 2> gpurun_out/r2d/cfg2.err
for f in gpurun_out/r2d/*.json; do python - "$f" <<'PY'
import json, sys
for l in open(sys.argv[1]):
    if l.startswith('{'):
        d = json.loads(l); e = d.get('e2e') or {}
        print(sys.argv[1], round(d['ms_per_step'], 3), '%.3g' % d['value'], d.get('frames_per_s'), 'e2e', e.get('value'), e.get('ms_per_step'), d.get('stages_ms'))
PY
done
