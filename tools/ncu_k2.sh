# ncu --set full of one K2 launch (cfg2 by default) -> gpurun_out/k2_<tag>.ncu-rep
cd $GRAFT_REPO_ROOT
CFG=${CFG:-cfg2}
TAG=${TAG:-new}
KREGEX=${KREGEX:-k2_}
timeout 900 ncu --set full --import-source on --clock-control none -k regex:$KREGEX --launch-skip 2 --launch-count 1 \
  -o gpurun_out/k2_${TAG}_${CFG} -f python tools/profile_frame.py --config $CFG --frames 4 > gpurun_out/ncu_k2_${TAG}_${CFG}.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_k2_${TAG}_${CFG}.log
