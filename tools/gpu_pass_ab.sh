#!/bin/bash
# Parent-pass floor A/B at s22/s24 ef16 and s26/s29 ef8 (variants given in $V).
cd ${GRAFT_REPO_ROOT:-.}
V=${V:-"libbflybfs.so libbflybfs_f16.so libbflybfs_f18.so libbflybfs.so libbflybfs_f16.so libbflybfs_f18.so"}
for c in "29 8" "26 8" "24 16" "22 16"; do set -- $c
SW_SCALE=$1 SW_EF=$2 SW_ROOTS=16 timeout 900 python tools/expand_sweep.py $V 2>&1 | grep "top-down parents=True" | sed "s/^/s$1 /; s/ exchange=.*//"
done
