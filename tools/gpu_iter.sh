#!/bin/bash
# One iteration: fast GPU tests, N=1 bench, BFS launch list, (optional) N=2 protocol run.
cd ${GRAFT_REPO_ROOT:-.}
timeout 1200 python -m pytest tests -q -x -m "gpu and not slow" --timeout=600 > gpurun_out/tq.log 2>&1
echo "tests rc=$?" >> gpurun_out/tq.log; tail -2 gpurun_out/tq.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench rc=$?" >> gpurun_out/bench.err
python - <<'PY'
import json
d=json.loads(open("gpurun_out/bench.json").read().strip().splitlines()[-1])
print({k: d.get(k) for k in ("value","bfs_ms_mean")}, "e2e", d["e2e"]["value"], "DO", d["direction_optimizing"]["value"], d["direction_optimizing"]["bfs_ms_mean"], "frac", d["roofline"]["frac"], "clocks", d["clocks"]["sm_mhz"], d["clocks"]["reasons"], "cpu", d["cpu_baseline"]["value"], d["cpu_baseline"]["levels_match_gpu"])
PY
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
ncu --metrics $M --clock-control none --csv --log-file gpurun_out/launch_td2.csv python tools/profile_bfs.py --runs 0 --parents 1 > /dev/null 2>&1
python tools/launches.py gpurun_out/launch_td2.csv 40 30 > gpurun_out/launch_td2.txt
tail -14 gpurun_out/launch_td2.txt
if [ -n "${N2:-}" ]; then
BFB_SHARED_GPU=1 BFB_DIST_BACKEND=gloo timeout 1200 python bench.py --gpus 2 --scale ${N2_SCALE:-26} --steps 2 --warmup 3 > gpurun_out/bench_n2.json 2> gpurun_out/bench_n2.err
echo "n2 rc=$?"; tail -c 1500 gpurun_out/bench_n2.json
fi
