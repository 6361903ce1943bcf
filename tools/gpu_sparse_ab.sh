#!/bin/bash
# Sparse-level threshold A/B (s29 ef8 and s24 ef16, 16 roots).
cd ${GRAFT_REPO_ROOT:-.}
SW_ROOTS=16 timeout 1500 python tools/expand_sweep.py libbflybfs.so libbflybfs_c24.so libbflybfs.so libbflybfs_c24.so 2>&1 | grep "parents=True" > gpurun_out/sp29.log
SW_SCALE=24 SW_EF=16 SW_ROOTS=16 timeout 900 python tools/expand_sweep.py libbflybfs.so libbflybfs_sp5.so libbflybfs_sp4.so libbflybfs.so libbflybfs_sp5.so libbflybfs_sp4.so 2>&1 | grep "parents=True" > gpurun_out/sp24.log
cat gpurun_out/sp29.log gpurun_out/sp24.log | sed 's/ exchange=.*//'
