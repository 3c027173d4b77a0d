# A/B of cache kernel variants (paper_2604_02586_b200/_lib/ab/<name>.so) with tools/cache_timing.py
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/cacheab
for c in ${CFGS:-cfg2 cfg5}; do
  timeout 300 python tools/cache_timing.py --config $c --frames 8 > gpurun_out/cacheab/base_$c.log 2>&1
  for v in ${VARIANTS}; do
    TS_LIB_PATH=$PWD/paper_2604_02586_b200/_lib/ab/$v.so timeout 300 python tools/cache_timing.py --config $c --frames 8 > gpurun_out/cacheab/${v}_$c.log 2>&1
  done
done
for f in gpurun_out/cacheab/*.log; do echo "$f: $(grep -o "'k2_raster_accumulate': [0-9.]*" $f | tail -1)"; done
