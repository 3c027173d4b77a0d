cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out/last
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/last/bench_cfg2.json 2> gpurun_out/last/bench_cfg2.err
timeout 600 python bench.py --config cfg5 --steps 20 --warmup 5 --no-cpu > gpurun_out/last/bench_cfg5.json 2> gpurun_out/last/bench_cfg5.err
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/last/smoke.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/last/smoke.txt
