cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -x -q -m "gpu and not slow" > gpurun_out/t5.log 2>&1
echo "tests rc=$?" >> gpurun_out/t5.log
BFB_SHARED_GPU=1 BFB_DIST_BACKEND=gloo timeout 900 python bench.py --gpus 2 --scale 24 --edge-factor 16 --steps 2 --warmup 3 > gpurun_out/b5n2.log 2> gpurun_out/b5n2.err
echo "bench2 rc=$?" >> gpurun_out/b5n2.err
tail -3 gpurun_out/t5.log
