mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/final_gputests.log 2>&1; echo "gputests rc=$?" >> gpurun_out/final_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/final_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/final_smoke.log
bash tools/run_profiles.sh > gpurun_out/run_profiles.log 2>&1
