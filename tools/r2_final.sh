# End-of-round pass at HEAD: GPU tests, smoke, bench lines (run_profiles.sh STAGE=bench) and the
# cfg2 / cfg5 ncu launch lists of whole frames.
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out/r02
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r02/gpu_tests.txt 2>&1; echo "gputests rc=$?" >> gpurun_out/r02/gpu_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02/smoke.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/r02/smoke.txt
STAGE=bench bash tools/run_profiles.sh > gpurun_out/r02/run_profiles_bench.log 2>&1
O=gpurun_out/r02
for c in cfg2 cfg5; do
  timeout 600 ncu --nvtx --nvtx-include "frame/" --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $O/launches_$c.csv python tools/profile_frame.py --config $c --frames 3 --lean > $O/ncu_launch_$c.log 2>&1
  python tools/summarize_ncu.py launches $O/launches_$c.csv > $O/launches_$c.txt 2>&1
  rm -f $O/launches_$c.csv
done
echo done
