#!/bin/bash
# Direction-switch threshold grid (alpha, beta), s29 ef8 and s24 ef16, 16 roots.
cd ${GRAFT_REPO_ROOT:-.}
L=libbflybfs.so
S="$L:SW_ALPHA=7,SW_BETA=64 $L:SW_ALPHA=14,SW_BETA=64 $L:SW_ALPHA=14,SW_BETA=24 $L:SW_ALPHA=10,SW_BETA=64 $L:SW_ALPHA=20,SW_BETA=64 $L:SW_ALPHA=14,SW_BETA=128 $L:SW_ALPHA=14,SW_BETA=32 $L:SW_ALPHA=7,SW_BETA=64 $L:SW_ALPHA=14,SW_BETA=64"
SW_ROOTS=16 timeout 1500 python tools/expand_sweep.py $S 2>&1 | grep optimizing | grep "parents=True" > gpurun_out/dogrid29.log
SW_SCALE=24 SW_EF=16 SW_ROOTS=16 timeout 900 python tools/expand_sweep.py $S 2>&1 | grep optimizing | grep "parents=True" > gpurun_out/dogrid24.log
cat gpurun_out/dogrid29.log gpurun_out/dogrid24.log | sed 's/ expand=.*bu_levels/ bu/'
