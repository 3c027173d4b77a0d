# Round-2 measurement pass on one B200 (run under gpurun); outputs in gpurun_out/r02_* (text and
# small files only: the ncu reports are summarised on the box and deleted, gpurun copies back at
# most 64 MiB).
#   bench lines (weak, every BASELINE config), the reference arm (cfg2), strong-scaling clips,
#   ncu launch lists of whole frames (cfg2, cfg5) and --set full captures of one whole frame
#   (cfg2, cfg5) plus K2 alone at cfg1/3/4 (roofline.traffic of every config).
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out/r02
O=gpurun_out/r02
STAGE=${STAGE:-all}
if [ $STAGE = all -o $STAGE = bench ]; then
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > $O/bench_reference_cfg2.json 2> $O/bench_reference_cfg2.err
for c in cfg2 cfg1 cfg3 cfg4 cfg5; do
  extra=""; [ $c != cfg2 ] && extra="--no-cpu"
  timeout 900 python bench.py --config $c --steps 20 --warmup 5 $extra > $O/bench_$c.json 2> $O/bench_$c.err
done
timeout 900 python bench.py --config cfg5 --clip-frames 8 --steps 3 --warmup 1 > $O/bench_cfg5_clip8.json 2> $O/bench_cfg5_clip8.err
timeout 900 python bench.py --config cfg4 --clip-frames 8 --steps 5 --warmup 2 > $O/bench_cfg4_clip8.json 2> $O/bench_cfg4_clip8.err
fi
if [ $STAGE = all -o $STAGE = ncu ]; then
for c in ${FRAME_CFGS:-cfg2 cfg5}; do
  timeout 600 ncu --nvtx --nvtx-include "frame/" --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $O/launches_$c.csv python tools/profile_frame.py --config $c --frames 3 > $O/ncu_launch_$c.log 2>&1
  python tools/summarize_ncu.py launches $O/launches_$c.csv > $O/launches_$c.txt 2>&1
  # one whole frame (the third one)
  timeout 1500 ncu --set full --clock-control none --nvtx --nvtx-include "frame/" \
    --launch-skip 70 --launch-count 35 -o /tmp/frame_$c -f python tools/profile_frame.py --config $c --frames 3 > $O/ncu_full_$c.log 2>&1
  python tools/summarize_ncu.py report /tmp/frame_$c.ncu-rep > $O/kernels_$c.txt 2>&1
  python tools/k2_traffic.py /tmp/frame_$c.ncu-rep $c "profiles/r02_kernels_$c.txt (ncu --set full --clock-control none of one whole $c frame via tools/profile_frame.py)" $O >> $O/ncu_full_$c.log 2>&1
done
for c in ${K2_CFGS:-cfg1 cfg3 cfg4}; do
  # K2 of the second timed frame (NVTX "frame" ranges: the tracker's dominant-mode launches of
  # the input generation are outside them)
  timeout 900 ncu --set full --clock-control none --nvtx --nvtx-include "frame/" -k regex:k2_raster \
    --launch-skip 1 --launch-count 1 -o /tmp/k2_$c -f python tools/profile_frame.py --config $c --frames 3 > $O/ncu_k2_$c.log 2>&1
  python tools/summarize_ncu.py report /tmp/k2_$c.ncu-rep > $O/k2_$c.txt 2>&1
  python tools/k2_traffic.py /tmp/k2_$c.ncu-rep $c "profiles/r02_k2_$c.txt (ncu --set full --clock-control none of K2 at $c via tools/profile_frame.py)" $O >> $O/ncu_k2_$c.log 2>&1
done
# K2 alone at cfg2 with source lines (small report kept for the per-line attribution)
timeout 900 ncu --set full --import-source on --clock-control none --nvtx --nvtx-include "frame/" -k regex:k2_raster \
  --launch-skip 1 --launch-count 1 -o $O/k2_cfg2 -f python tools/profile_frame.py --config cfg2 --frames 3 > $O/ncu_k2_cfg2.log 2>&1
fi
if [ $STAGE = all -o $STAGE = clip ]; then
# clip mode with the contribution cache: launch list of cache builds ("build") and cached frames
# ("frame"), and one --set full capture of a cached cfg5 frame
for c in ${CLIP_CFGS:-cfg4 cfg5}; do
  timeout 600 ncu --nvtx --nvtx-include "build/" --nvtx-include "frame/" --metrics gpu__time_duration.sum \
    --clock-control none --csv --log-file $O/clip_launches_$c.csv python tools/cache_timing.py --config $c \
    --frames 8 --passes 1,1 > $O/ncu_clip_launch_$c.log 2>&1
  python tools/summarize_ncu.py launches $O/clip_launches_$c.csv > $O/clip_launches_$c.txt 2>&1
done
timeout 900 ncu --set full --clock-control none --nvtx --nvtx-include "frame/" -k regex:"k23_cached|k3_merge|k4_fuse" --launch-skip 6 --launch-count 4 \
  -o /tmp/clip_cfg5 -f python tools/cache_timing.py --config cfg5 --frames 8 --passes 1,1 > $O/ncu_clip_full_cfg5.log 2>&1
python tools/summarize_ncu.py report /tmp/clip_cfg5.ncu-rep > $O/clip_kernels_cfg5.txt 2>&1
timeout 900 python bench.py --config cfg5 --clip-frames 8 --steps 3 --warmup 3 > $O/bench_cfg5_clip8.json 2> $O/bench_cfg5_clip8.err
timeout 900 python bench.py --config cfg4 --clip-frames 8 --steps 5 --warmup 3 > $O/bench_cfg4_clip8.json 2> $O/bench_cfg4_clip8.err
timeout 900 python bench.py --config cfg5 --clip-frames 8 --no-cache --steps 3 --warmup 3 > $O/bench_cfg5_clip8_nocache.json 2> $O/bench_cfg5_clip8_nocache.err
fi
du -sh $O
echo done
