# launch list (gpu__time_duration) of one frame's kernels for a config -> gpurun_out/launches_<tag>_<cfg>.csv
cd $GRAFT_REPO_ROOT
CFG=${CFG:-cfg5}
TAG=${TAG:-r2}
timeout 900 ncu --nvtx --nvtx-include "frame/" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,sm__warps_active.avg.per_cycle_active --clock-control none --csv --launch-skip 40 --launch-count 40 \
  --log-file gpurun_out/launches_${TAG}_${CFG}.csv python tools/profile_frame.py --config $CFG --frames 3 > gpurun_out/ncu_launch_${TAG}_${CFG}.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_launch_${TAG}_${CFG}.log
