#!/bin/bash
# Un-permute A/B (default vs cp.async perm prefetch): ncu time in one s29 BFS,
# interleaved sweep, parity tests on the variant.
cd ${GRAFT_REPO_ROOT:-.}
LIBS=${LIBS:-"libbflybfs.so libbflybfs_os.so"}
for L in $LIBS; do
BFB_LIB=$L ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_output --csv python tools/profile_bfs.py --runs 0 --parents 1 2>/dev/null | grep -E "gpu__time|dram__" | sed "s/^/$L /" | cut -c1-30,160-
done
SW_ROOTS=16 timeout 1500 python tools/expand_sweep.py $LIBS $LIBS 2>&1 | grep "parents=True" | sed 's/ exchange=.*//'
BFB_LIB=${TLIB:-libbflybfs_os.so} timeout 900 python -m pytest tests/test_gpu_readout.py tests/test_gpu_bfs.py tests/test_gpu_parity.py -q -x -m "gpu and not slow" > gpurun_out/to.log 2>&1; echo "variant tests rc=$?"; tail -1 gpurun_out/to.log
