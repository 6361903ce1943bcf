ncu --set full --import-source on --clock-control none -k regex:k_commit_write -s 5 -c 1 -f -o gpurun_out/cw5 python tools/profile_bfs.py --runs 0 --parents 1 > gpurun_out/prof_c.log 2>&1
