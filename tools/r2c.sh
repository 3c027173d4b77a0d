# cache A/B on the GPU: cache tests, per-stage timing, one ncu capture of the cached kernel
mkdir -p gpurun_out/r2c
timeout 900 python -m pytest tests -m gpu -x -q -k "cache or pipeline" > gpurun_out/r2c/tests.log 2>&1; echo tests=$?
for c in ${CONFIGS:-cfg2 cfg5}; do timeout 300 python tools/cache_timing.py --config $c --frames 8 > gpurun_out/r2c/timing_$c.log 2>&1; done
if [ -n "$NCU" ]; then
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k23_cached -c 1 \
    -o gpurun_out/r2c/k2c python tools/cache_timing.py --config cfg2 --frames 2 > gpurun_out/r2c/ncu.log 2>&1
  python tools/summarize_ncu.py report gpurun_out/r2c/k2c.ncu-rep > gpurun_out/r2c/k2c_summary.txt 2>&1
fi
tail -n 4 gpurun_out/r2c/*.log gpurun_out/r2c/*.txt
