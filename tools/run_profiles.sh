mkdir -p gpurun_out
for c in cfg2 cfg1 cfg3 cfg4 cfg5; do
  extra=""; [ $c != cfg2 ] && extra="--no-cpu"
  timeout 600 python bench.py --config $c $extra > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
done
timeout 400 python bench.py --impl reference > gpurun_out/bench_reference_cfg2.json 2> gpurun_out/bench_reference_cfg2.err
timeout 300 ncu --nvtx --nvtx-include "frame/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/profile_frame.py --frames 2 > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none --nvtx --nvtx-include "frame/" --launch-skip 31 --launch-count 31 -o gpurun_out/frame_cfg2 -f python tools/profile_frame.py --frames 2 > gpurun_out/ncu_full.log 2>&1
echo done
