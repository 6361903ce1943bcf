#!/bin/bash
# Quick GPU check: the fast GPU tests, then the default bench line.
cd ${GRAFT_REPO_ROOT:-.}
timeout 1200 python -m pytest tests -q -x -m "gpu and not slow" --timeout=600 > gpurun_out/tq.log 2>&1
echo "tests rc=$?" >> gpurun_out/tq.log
timeout 900 python bench.py ${BENCH_ARGS:-} > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench rc=$?" >> gpurun_out/bench.err
tail -3 gpurun_out/tq.log; tail -2 gpurun_out/bench.err
python - <<'PY'
import json
d=json.loads(open("gpurun_out/bench.json").read().strip().splitlines()[-1])
print({k: d.get(k) for k in ("value","bfs_ms_mean","ms_per_step")}, "e2e", d["e2e"]["value"], "DO", d["direction_optimizing"]["value"], "frac", d["roofline"]["frac"], "clocks", d["clocks"])
PY
