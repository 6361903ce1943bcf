cd $GRAFT_REPO_ROOT
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1200 python -m pytest tests/test_gpu_acceptance.py tests/test_gpu_bfs.py -q -m gpu -x --durations=40 -k "acceptance or deep or tiny or spec or errors" > gpurun_out/t_small.log 2>&1
echo "rc=$?" >> gpurun_out/t_small.log
tail -50 gpurun_out/t_small.log; cat gpurun_out/smoke.log
