#!/bin/bash
# Tuning sweep over library variants (tools/expand_sweep.py), results in gpurun_out/sweep.log
cd ${GRAFT_REPO_ROOT:-.}
SW_ROOTS=${SW_ROOTS:-12} timeout ${SWEEP_TIMEOUT:-2400} python tools/expand_sweep.py $SWEEP > gpurun_out/sweep.log 2>&1
cat gpurun_out/sweep.log
