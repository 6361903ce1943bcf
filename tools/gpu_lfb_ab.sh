#!/bin/bash
# Level materialisation A/B: ncu time of the byte-form kernel in one s29 BFS per
# library, then the interleaved sweep, then the GPU tests on the default build.
cd ${GRAFT_REPO_ROOT:-.}
LIBS=${LIBS:-"libbflybfs.so libbflybfs_thr.so libbflybfs_thr8.so"}
for L in $LIBS; do
BFB_LIB=$L ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_levels --csv python tools/profile_bfs.py --runs 0 --parents 1 2>/dev/null | grep -E "gpu__time" | sed "s/^/$L /" | cut -c1-40,150-
done
SW_ROOTS=16 timeout 1500 python tools/expand_sweep.py $LIBS $LIBS 2>&1 | grep "parents=True" | sed 's/ exchange=.*//'
timeout 1500 python -m pytest tests -q -x -m "gpu and not slow" --timeout=900 > gpurun_out/tq.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/tq.log
