# A/B of the depth-key width (ab/d28.so: up to 28 quantised depth bits) vs the in-tree library,
# updates-only frames (the bench's outputs), then the GPU suite on the in-tree library and on d28.
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
for c in ${CFGS:-cfg2 cfg5}; do
for r in 1 2; do
TS_LIB_PATH=$PWD/paper_2604_02586_b200/_lib/ab/d28.so timeout 300 python tools/profile_frame.py --config $c --frames 10 --lean > gpurun_out/d28ab_d28_${c}_$r.log 2>&1
timeout 300 python tools/profile_frame.py --config $c --frames 10 --lean > gpurun_out/d28ab_new_${c}_$r.log 2>&1
done
done
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/d28ab_gputests_new.log 2>&1; echo rc=$? >> gpurun_out/d28ab_gputests_new.log
TS_LIB_PATH=$PWD/paper_2604_02586_b200/_lib/ab/d28.so timeout 1200 python -m pytest tests -m gpu -x -q -k "scale or edge or parity" > gpurun_out/d28ab_gputests_d28.log 2>&1; echo rc=$? >> gpurun_out/d28ab_gputests_d28.log
