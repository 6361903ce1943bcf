#!/bin/bash
# Extra ncu captures: the dense write pass (level 2), the first bottom-up
# level, the level materialisation (SASS stall attribution via ncu_hot_sass.py)
cd ${GRAFT_REPO_ROOT:-.}
P="python tools/profile_bfs.py --runs 0 --parents 1"
FULL="ncu --set full --import-source on --clock-control none -f"
$FULL -k regex:k_commit_write -s 1 -c 1 -o gpurun_out/cw2 $P > /dev/null 2>&1
$FULL -k regex:k_bottom_up -s 0 -c 1 -o gpurun_out/bu $P --direction optimizing > /dev/null 2>&1
$FULL -k regex:k_levels -c 1 -o gpurun_out/lfb $P > /dev/null 2>&1
for r in cw2 bu lfb; do python tools/ncu_summary.py gpurun_out/$r.ncu-rep > gpurun_out/$r.txt 2>&1; python tools/ncu_hot_sass.py gpurun_out/$r.ncu-rep 12 >> gpurun_out/$r.txt 2>&1; done
cat gpurun_out/cw2.txt gpurun_out/bu.txt gpurun_out/lfb.txt
