# A/B of library builds: TS_LIB_PATH=paper_2604_02586_b200/_lib/ab/<name>.so vs the in-tree one
cd $GRAFT_REPO_ROOT
for c in ${CFGS:-cfg2 cfg5}; do
for v in ${VARIANTS:-old}; do
TS_LIB_PATH=$PWD/paper_2604_02586_b200/_lib/ab/$v.so timeout 300 python tools/profile_frame.py --config $c --frames 10 > gpurun_out/r2_libab_${v}_$c.log 2>&1
done
timeout 300 python tools/profile_frame.py --config $c --frames 10 > gpurun_out/r2_libab_new_$c.log 2>&1
done
