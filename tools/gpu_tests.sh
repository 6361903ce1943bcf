#!/bin/bash
# Full GPU suite with per-test durations (gpurun_out/tests.log).
cd ${GRAFT_REPO_ROOT:-.}
timeout ${TEST_TIMEOUT:-2700} python -m pytest tests -q -m gpu -rs --timeout=1200 --durations=60 > gpurun_out/tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/tests.log
tail -75 gpurun_out/tests.log
