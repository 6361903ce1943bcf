#!/bin/bash
# A/B of two library builds (tools/expand_sweep.py, interleaved), then the fast GPU tests.
cd ${GRAFT_REPO_ROOT:-.}
A=${A:-libbflybfs_prev.so}; B=${B:-libbflybfs.so}
SW_ROOTS=${SW_ROOTS:-16} timeout 900 python tools/expand_sweep.py $A $B $A $B > gpurun_out/sweep.log 2>&1
grep "parents=True" gpurun_out/sweep.log
if [ -z "${NOTEST:-}" ]; then
timeout 1500 python -m pytest tests -q -x -m "gpu and not slow" --timeout=900 > gpurun_out/tq.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/tq.log
fi
