# A/B of the K2 accumulate kernels (TS_K2_LEGACY=1: the pixel-owned loop) + the GPU suite
cd $GRAFT_REPO_ROOT
for c in ${CFGS:-cfg2 cfg5}; do
TS_K2_LEGACY=1 timeout 300 python tools/profile_frame.py --config $c --frames 10 > gpurun_out/r2_k2ab_legacy_$c.log 2>&1
timeout 300 python tools/profile_frame.py --config $c --frames 10 > gpurun_out/r2_k2ab_new_$c.log 2>&1
done
if [ -z "$NOTESTS" ]; then
timeout 1500 python -m pytest tests -m gpu -q -x -rs ${TESTK:+-k "$TESTK"} > gpurun_out/r2_gputests_k2b.log 2>&1; echo rc=$? >> gpurun_out/r2_gputests_k2b.log
fi
