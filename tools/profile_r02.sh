#!/bin/bash
# Round-2 profile captures (gpurun): launch lists of one s29 BFS (top-down and
# direction-optimizing, levels read out) and ncu --set full captures of the
# densest top-down level's expand, its commit count pass (parent pass) and a
# write pass.  Summaries go to profiles/ via tools/launches.py / ncu_summary.py.
set -u
cd ${GRAFT_REPO_ROOT:-.}
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
P="python tools/profile_bfs.py --runs 0 --parents 1"
FULL="ncu --set full --import-source on --clock-control none -f"
ncu --metrics $M --clock-control none --csv --log-file gpurun_out/launch_td.csv $P --levels 1 > gpurun_out/prof_td.log 2>&1
ncu --metrics $M --clock-control none --csv --log-file gpurun_out/launch_do.csv $P --levels 1 --direction optimizing > gpurun_out/prof_do.log 2>&1
python tools/launches.py gpurun_out/launch_td.csv 0 30 > gpurun_out/launch_td.txt
python tools/launches.py gpurun_out/launch_do.csv 0 30 > gpurun_out/launch_do.txt
$FULL -k regex:k_expand_w -s ${EXP_SKIP:-3} -c 1 -o gpurun_out/expw $P > gpurun_out/prof_e.log 2>&1
$FULL -k regex:k_commit_count -s ${CC_SKIP:-3} -c 1 -o gpurun_out/ccp $P > gpurun_out/prof_cc.log 2>&1
$FULL -k regex:k_commit_write -s ${CW_SKIP:-5} -c 1 -o gpurun_out/cw $P > gpurun_out/prof_cw.log 2>&1
for r in expw ccp cw; do python tools/ncu_summary.py gpurun_out/$r.ncu-rep > gpurun_out/$r.txt 2>&1; done
cat gpurun_out/launch_td.txt gpurun_out/expw.txt
