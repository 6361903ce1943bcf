#!/bin/bash
# The C2 (s24 ef16) bench line and the N=2 protocol line (2 ranks sharing one GPU).
cd ${GRAFT_REPO_ROOT:-.}
timeout 900 python bench.py --scale 24 --edge-factor 16 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
echo "c2 rc=$?"
BFB_SHARED_GPU=1 BFB_DIST_BACKEND=gloo timeout 1200 python bench.py --gpus 2 --scale 26 --steps 2 --warmup 3 > gpurun_out/bench_n2.json 2> gpurun_out/bench_n2.err
echo "n2 rc=$?"; tail -c 300 gpurun_out/bench_c2.json; tail -c 300 gpurun_out/bench_n2.json
