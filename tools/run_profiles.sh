# Round-2 measurement pass on one B200 (run under gpurun); outputs in gpurun_out/r02_*.
#   bench lines (weak, every BASELINE config), the reference arm (cfg2), strong-scaling clips,
#   ncu launch lists of whole frames (cfg2, cfg5) and --set full captures of one whole frame
#   (cfg2, cfg5) plus K2 alone at cfg1/3/4 (roofline.traffic of every config).
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
O=gpurun_out
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > $O/r02_bench_reference_cfg2.json 2> $O/r02_bench_reference_cfg2.err
for c in cfg2 cfg1 cfg3 cfg4 cfg5; do
  extra=""; [ $c != cfg2 ] && extra="--no-cpu"
  timeout 900 python bench.py --config $c --steps 20 --warmup 5 $extra > $O/r02_bench_$c.json 2> $O/r02_bench_$c.err
done
timeout 900 python bench.py --config cfg5 --clip-frames 8 --steps 3 --warmup 1 > $O/r02_bench_cfg5_clip8.json 2> $O/r02_bench_cfg5_clip8.err
timeout 900 python bench.py --config cfg4 --clip-frames 8 --steps 5 --warmup 2 > $O/r02_bench_cfg4_clip8.json 2> $O/r02_bench_cfg4_clip8.err
for c in cfg2 cfg5; do
  timeout 600 ncu --nvtx --nvtx-include "frame/" --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $O/r02_launches_$c.csv python tools/profile_frame.py --config $c --frames 3 > $O/r02_ncu_launch_$c.log 2>&1
  # one whole frame (the third: launches 2F..3F-1 of the frame ranges)
  timeout 1500 ncu --set full --import-source on --clock-control none --nvtx --nvtx-include "frame/" \
    --launch-skip 70 --launch-count 35 -o $O/r02_frame_$c -f python tools/profile_frame.py --config $c --frames 3 > $O/r02_ncu_full_$c.log 2>&1
done
for c in cfg1 cfg3 cfg4; do
  timeout 900 ncu --set full --clock-control none -k regex:k2_raster --launch-skip 2 --launch-count 1 \
    -o $O/r02_k2_$c -f python tools/profile_frame.py --config $c --frames 4 > $O/r02_ncu_k2_$c.log 2>&1
done
echo done
