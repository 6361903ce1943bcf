#!/bin/bash
# Direction-switch threshold sweep (s29, 16 roots) and the C2 / N=2-protocol
# bench lines with the current build.
cd ${GRAFT_REPO_ROOT:-.}
L=libbflybfs.so
SW_ROOTS=16 timeout 1500 python tools/expand_sweep.py $L:SW_ALPHA=5 $L:SW_ALPHA=3 $L:SW_ALPHA=4 $L:SW_ALPHA=7 \
  $L:SW_ALPHA=5,SW_BETA=256 $L:SW_ALPHA=5,SW_BETA=4096 $L:SW_ALPHA=5,SW_BETA=1e9 $L:SW_ALPHA=5 2>&1 | grep optimizing | grep "parents=True" > gpurun_out/dosweep.log
cat gpurun_out/dosweep.log
SW_SCALE=24 SW_EF=16 SW_ROOTS=16 timeout 600 python tools/expand_sweep.py $L:SW_ALPHA=5 $L:SW_ALPHA=3 $L:SW_ALPHA=8 2>&1 | grep optimizing | grep "parents=True" > gpurun_out/dosweep24.log
cat gpurun_out/dosweep24.log
timeout 900 python bench.py --scale 24 --edge-factor 16 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
BFB_SHARED_GPU=1 BFB_DIST_BACKEND=gloo timeout 1200 python bench.py --gpus 2 --scale 26 --steps 2 --warmup 3 > gpurun_out/bench_n2.json 2> gpurun_out/bench_n2.err
echo "n2 rc=$?"; tail -c 400 gpurun_out/bench_c2.json; tail -c 400 gpurun_out/bench_n2.json
