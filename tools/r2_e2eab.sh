# e2e modes with the in-tree library vs a variant (TS_LIB_PATH)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/e2eab
for rep in 1 2; do
for v in ${VARIANTS:-scalar} new; do
  if [ $v = new ]; then L=""; else L=$PWD/paper_2604_02586_b200/_lib/ab/$v.so; fi
  TS_LIB_PATH=$L timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read()); e=d['e2e']
print('$v', round(d['ms_per_step'],3), {k: round(e[k]['ms_per_step'],3) for k in ('rect_copy','zero_copy','auto','full_copy')}, d['stage_ms']['k2_raster_accumulate'])"
done; done
