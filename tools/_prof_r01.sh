M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
ncu --metrics $M --clock-control none --csv --log-file gpurun_out/launch_td.csv python tools/profile_bfs.py --runs 0 --parents 1 --levels 1 > gpurun_out/prof_td.log 2>&1
ncu --metrics $M --clock-control none --csv --log-file gpurun_out/launch_do.csv python tools/profile_bfs.py --runs 0 --parents 1 --levels 1 --direction optimizing > gpurun_out/prof_do.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_expand_w -s 3 -c 1 -f -o gpurun_out/expw4 python tools/profile_bfs.py --runs 0 --parents 1 > gpurun_out/prof_e.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_commit_write -s 2 -c 1 -f -o gpurun_out/cw4 python tools/profile_bfs.py --runs 0 --parents 1 > gpurun_out/prof_c.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_bottom_up -s 0 -c 1 -f -o gpurun_out/bu4 python tools/profile_bfs.py --runs 0 --parents 1 --direction optimizing > gpurun_out/prof_b.log 2>&1
ls -la gpurun_out/
