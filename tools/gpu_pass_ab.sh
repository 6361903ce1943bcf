#!/bin/bash
# Parent-pass floor A/B (old = no floor) at s22/s24 ef16 and s26/s29 ef8, then the fast GPU tests.
cd ${GRAFT_REPO_ROOT:-.}
V="libbflybfs_old.so libbflybfs.so libbflybfs_old.so libbflybfs.so"
for c in "29 8" "26 8" "24 16" "22 16"; do set -- $c
SW_SCALE=$1 SW_EF=$2 SW_ROOTS=16 timeout 900 python tools/expand_sweep.py $V 2>&1 | grep "top-down parents=True" | sed "s/^/s$1 /; s/ exchange=.*//"
done
timeout 1500 python -m pytest tests -q -x -m "gpu and not slow" --timeout=900 > gpurun_out/tq.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/tq.log
