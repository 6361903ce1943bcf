#!/bin/bash
# e2e A/B: read-out destinations on 2 MB pages (BFB_HOST_HUGE=1) vs cudaHostAlloc.
cd ${GRAFT_REPO_ROOT:-.}
cat /sys/kernel/mm/transparent_hugepage/enabled /sys/kernel/mm/transparent_hugepage/defrag
for h in 0 1 0 1; do echo -n "huge=$h "; BFB_HOST_HUGE=$h timeout 600 python tools/e2e_ab.py 2>&1 | tail -1; done
BFB_HOST_HUGE=1 timeout 600 python -m pytest tests/test_gpu_readout.py -q -x 2>&1 | tail -1
