# ncu --set full of the K1 kernels (depth bounds, projection + keys, bbox union, emit, tie repair)
# of one cfg5 and one cfg2 frame (updates-only path, as the bench)
cd ${GRAFT_REPO_ROOT:-.}
O=gpurun_out/r02k1; mkdir -p $O
for c in cfg5 cfg2; do
timeout 900 ncu --set full --clock-control none --nvtx --nvtx-include "frame/" -k regex:"k1_" \
  --launch-skip 7 --launch-count 7 -o /tmp/k1_$c -f python tools/profile_frame.py --config $c --frames 3 --lean > $O/ncu_k1_$c.log 2>&1
python tools/summarize_ncu.py report /tmp/k1_$c.ncu-rep > $O/k1_$c.txt 2>&1
done
echo done
