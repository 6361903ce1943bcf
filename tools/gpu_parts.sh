#!/bin/bash
# Multi-part single-GPU A/B (tools/expand_sweep.py with SW_PARTS), then the multi-node tests.
cd ${GRAFT_REPO_ROOT:-.}
A=${A:-libbflybfs_prev.so}; B=${B:-libbflybfs.so}
for P in ${PARTS:-8 2}; do SW_PARTS=$P SW_ROOTS=8 timeout 600 python tools/expand_sweep.py $A $B 2>&1 | grep "parents=True" | sed "s/^/P=$P /"; done
if [ -z "${NOTEST:-}" ]; then
timeout 1500 python -m pytest tests -q -x -m gpu --timeout=900 -k "${TESTK:-dist or acceptance or sweep or config3 or config4 or golden}" > gpurun_out/tp.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/tp.log
fi
