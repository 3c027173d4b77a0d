# driver-like bench runs: reference arm then ours (cfg2), plus cfg5 clip mode at world 1
cd $GRAFT_REPO_ROOT
( time timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 ) > gpurun_out/r2_bench_ref.json 2> gpurun_out/r2_bench_ref.err
( time timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 ) > gpurun_out/r2_bench_cfg2.json 2> gpurun_out/r2_bench_cfg2.err
timeout 900 python bench.py --config cfg5 --clip-frames 8 --steps 3 --warmup 1 > gpurun_out/r2_bench_cfg5_clip8.json 2> gpurun_out/r2_bench_cfg5_clip8.err
