# A/B of a variant library (ab/${VAR}.so) vs the in-tree one, updates-only frames, then the GPU
# updates-only frames (the bench's outputs), then the GPU suite on the in-tree library and on $VAR.
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
for c in ${CFGS:-cfg2 cfg5}; do
for r in 1 2; do
TS_LIB_PATH=$PWD/paper_2604_02586_b200/_lib/ab/${VAR}.so timeout 300 python tools/profile_frame.py --config $c --frames 10 --lean > gpurun_out/${VAR}ab_${VAR}_${c}_$r.log 2>&1
timeout 300 python tools/profile_frame.py --config $c --frames 10 --lean > gpurun_out/${VAR}ab_new_${c}_$r.log 2>&1
done
done
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/${VAR}ab_gputests_new.log 2>&1; echo rc=$? >> gpurun_out/${VAR}ab_gputests_new.log
TS_LIB_PATH=$PWD/paper_2604_02586_b200/_lib/ab/${VAR}.so timeout 1200 python -m pytest tests -m gpu -x -q -k "scale or edge or parity" > gpurun_out/${VAR}ab_gputests_${VAR}.log 2>&1; echo rc=$? >> gpurun_out/${VAR}ab_gputests_${VAR}.log
