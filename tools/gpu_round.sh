#!/bin/bash
# One gpurun call: full GPU test suite, default bench line, reference arm,
# launch list of one s29 BFS.  Everything lands in gpurun_out/.
set -u
cd ${GRAFT_REPO_ROOT:-.}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout ${TEST_TIMEOUT:-2400} python -m pytest tests -q -m gpu -rs --durations=25 > gpurun_out/tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/tests.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench rc=$?" >> gpurun_out/bench.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
echo "ref rc=$?" >> gpurun_out/bench_ref.err
tail -3 gpurun_out/tests.log; cat gpurun_out/bench.json gpurun_out/bench_ref.json
