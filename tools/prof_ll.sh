cd $GRAFT_REPO_ROOT
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
ncu --metrics $M --clock-control none --csv --log-file gpurun_out/launch_td2.csv python tools/profile_bfs.py --runs 0 --parents 1 > /dev/null 2>&1
python tools/launches.py gpurun_out/launch_td2.csv 40 30 > gpurun_out/launch_td2.txt
ncu --set full --import-source on --clock-control none -f -k regex:k_output -c 1 -o gpurun_out/kout python tools/profile_bfs.py --runs 0 --parents 1 > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/kout.ncu-rep > gpurun_out/kout.txt
cat gpurun_out/launch_td2.txt gpurun_out/kout.txt
