#!/bin/bash
# Level materialisation A/B: ncu time of the byte-form kernel in one s29 BFS per
# library, the interleaved sweep, then the parity tests on $TLIB.
cd ${GRAFT_REPO_ROOT:-.}
LIBS=${LIBS:-"libbflybfs.so libbflybfs_xp.so"}
for L in $LIBS; do
BFB_LIB=$L ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_levels --csv python tools/profile_bfs.py --runs 0 --parents 1 2>/dev/null | grep -E "gpu__time" | sed "s/^/$L /" | cut -c1-30,200-
done
SW_ROOTS=16 timeout 1500 python tools/expand_sweep.py $LIBS $LIBS 2>&1 | grep "parents=True" | sed 's/ exchange=.*//'
BFB_LIB=${TLIB:-libbflybfs_xp.so} timeout 900 python -m pytest tests/test_gpu_readout.py tests/test_gpu_bfs.py tests/test_gpu_parity.py -q -x -m "gpu and not slow" > gpurun_out/tx.log 2>&1; echo "variant tests rc=$?"; tail -1 gpurun_out/tx.log
