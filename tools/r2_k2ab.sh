cd $GRAFT_REPO_ROOT
for c in cfg2 cfg5; do
TS_K2_LEGACY=1 timeout 300 python tools/profile_frame.py --config $c --frames 10 > gpurun_out/r2_k2ab_legacy_$c.log 2>&1
timeout 300 python tools/profile_frame.py --config $c --frames 10 > gpurun_out/r2_k2ab_new_$c.log 2>&1
done
timeout 1500 python -m pytest tests -m gpu -q -x -rs > gpurun_out/r2_gputests_k2b.log 2>&1; echo rc=$? >> gpurun_out/r2_gputests_k2b.log
