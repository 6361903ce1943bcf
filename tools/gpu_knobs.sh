#!/bin/bash
# Thin-level and parent-pass threshold variants vs the default (s29 ef8 and s24 ef16, 16 roots).
cd ${GRAFT_REPO_ROOT:-.}
V="libbflybfs.so libbflybfs_t12.so libbflybfs_t14.so libbflybfs_ps10.so libbflybfs_ps14.so libbflybfs.so"
SW_ROOTS=16 timeout 1500 python tools/expand_sweep.py $V 2>&1 | grep "parents=True" > gpurun_out/kn29.log
SW_SCALE=24 SW_EF=16 SW_ROOTS=16 timeout 900 python tools/expand_sweep.py $V $V 2>&1 | grep "parents=True" > gpurun_out/kn24.log
cat gpurun_out/kn29.log gpurun_out/kn24.log | sed 's/ exchange=.*//'
