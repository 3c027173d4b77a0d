cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/e_gputests.log 2>&1; echo "gputests rc=$?" >> gpurun_out/e_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/e_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/e_smoke.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/e_bench_cfg2.json 2> gpurun_out/e_bench_cfg2.err; echo "bench rc=$?" >> gpurun_out/e_bench_cfg2.err
