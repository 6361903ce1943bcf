#!/bin/bash
# GPU suite (FULL=1: every gpu test, else the fast ones) and the C2 (s24 ef16) bench line.
cd ${GRAFT_REPO_ROOT:-.}
SEL="gpu and not slow"; [ -n "${FULL:-}" ] && SEL="gpu"
timeout 2400 python -m pytest tests -q -m "$SEL" -rs --timeout=1200 --durations=60 > gpurun_out/tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/tests.log
timeout 900 python bench.py --scale 24 --edge-factor 16 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
tail -2 gpurun_out/tests.log; tail -c 300 gpurun_out/bench_c2.json
