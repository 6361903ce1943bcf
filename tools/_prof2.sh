ncu --set full --import-source on --clock-control none -k regex:k_levels_from_bits -c 1 -f -o gpurun_out/lfb4 python tools/profile_bfs.py --runs 0 --parents 1 > gpurun_out/prof_l.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_commit_count -s 2 -c 1 -f -o gpurun_out/cc4 python tools/profile_bfs.py --runs 0 --parents 1 > gpurun_out/prof_cc.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_commit_count -s 5 -c 1 -f -o gpurun_out/cc5 python tools/profile_bfs.py --runs 0 --parents 1 > gpurun_out/prof_cc5.log 2>&1
