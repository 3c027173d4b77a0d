# A/B of the K3 split (TS_K3_SPLIT=0: one thread per gv over all gvs) on cfg2 / cfg5
cd $GRAFT_REPO_ROOT
for c in ${CFGS:-cfg2 cfg5}; do
TS_K3_SPLIT=0 timeout 300 python tools/profile_frame.py --config $c --frames 10 > gpurun_out/r2_k3ab_old_$c.log 2>&1
timeout 300 python tools/profile_frame.py --config $c --frames 10 > gpurun_out/r2_k3ab_new_$c.log 2>&1
done
