# A/B of two library builds: TS_LIB_PATH=paper_2604_02586_b200/_lib/ab/old.so vs the in-tree one
cd $GRAFT_REPO_ROOT
for c in ${CFGS:-cfg2 cfg5}; do
TS_LIB_PATH=$PWD/paper_2604_02586_b200/_lib/ab/old.so timeout 300 python tools/profile_frame.py --config $c --frames 10 > gpurun_out/r2_libab_old_$c.log 2>&1
timeout 300 python tools/profile_frame.py --config $c --frames 10 > gpurun_out/r2_libab_new_$c.log 2>&1
done
