#!/bin/bash
# Launch lists (ncu, serialised) of one s24 ef16 BFS, top-down and direction-optimizing.
cd ${GRAFT_REPO_ROOT:-.}
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
for d in top-down optimizing; do
ncu --metrics $M --clock-control none --csv --log-file gpurun_out/l24_$d.csv python tools/profile_bfs.py --scale 24 --edge-factor 16 --runs 1 --parents 1 --direction $d > gpurun_out/p24_$d.log 2>&1
python tools/launches.py gpurun_out/l24_$d.csv 0 0 > gpurun_out/l24_$d.txt
done
python tools/profile_bfs.py --scale 24 --edge-factor 16 --runs 3 --parents 1
