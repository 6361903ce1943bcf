#!/bin/bash
# Round profile captures (run on the GPU box via gpurun; writes gpurun_out/):
#   launch lists of one s29 BFS (top-down and direction-optimizing, levels
#   read out) and one ncu --set full capture per hot kernel.  Summaries for
#   profiles/ are made here afterwards with tools/launches.py,
#   tools/ncu_summary.py and tools/ncu_hot.py.
set -u
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
P="python tools/profile_bfs.py --runs 0 --parents 1"
FULL="ncu --set full --import-source on --clock-control none -f"
ncu --metrics $M --clock-control none --csv --log-file gpurun_out/launch_td.csv $P --levels 1 > gpurun_out/prof_td.log 2>&1
ncu --metrics $M --clock-control none --csv --log-file gpurun_out/launch_do.csv $P --levels 1 --direction optimizing > gpurun_out/prof_do.log 2>&1
# densest top-down level (4th expand launch), its commit with the parent pass
# (4th count launch), the write pass after the level-2 expand (6th write
# launch: two builds are launched per level), the first bottom-up level and
# the level materialisation
$FULL -k regex:k_expand_w -s 3 -c 1 -o gpurun_out/expw $P > gpurun_out/prof_e.log 2>&1
$FULL -k regex:k_commit_count -s 3 -c 1 -o gpurun_out/ccp $P > gpurun_out/prof_cc.log 2>&1
$FULL -k regex:k_commit_write -s 5 -c 1 -o gpurun_out/cw $P > gpurun_out/prof_cw.log 2>&1
$FULL -k regex:k_bottom_up -s 0 -c 1 -o gpurun_out/bu $P --direction optimizing > gpurun_out/prof_bu.log 2>&1
$FULL -k regex:k_levels_from_bits -c 1 -o gpurun_out/lfb $P > gpurun_out/prof_lfb.log 2>&1
ls -la gpurun_out/
