cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -x -q -m "gpu and not slow" > gpurun_out/t4.log 2>&1
echo "tests rc=$?" >> gpurun_out/t4.log
timeout 600 python bench.py --steps 2 --warmup 2 --cpu-roots 0 > gpurun_out/b4.log 2> gpurun_out/b4.err
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 900 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/launch4_td.csv python tools/profile_bfs.py --runs 1 --parents 1 --levels 0 > gpurun_out/prof4.log 2>&1
timeout 900 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/launch4_do.csv python tools/profile_bfs.py --runs 1 --parents 1 --levels 0 --direction optimizing > gpurun_out/prof4do.log 2>&1
tail -3 gpurun_out/t4.log
