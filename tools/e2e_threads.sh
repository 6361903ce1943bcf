#!/bin/bash
# e2e breakdown (tools/e2e_probe.py) for several read-out thread counts
cd ${GRAFT_REPO_ROOT:-.}
nproc; lscpu | grep -E "Model name|Socket|NUMA node|Thread|Core" | head -8
for t in 16 8 32; do echo "BFB_HOST_THREADS=$t"; BFB_HOST_THREADS=$t timeout 300 python tools/e2e_probe.py 29 2>&1 | tail -4; done
