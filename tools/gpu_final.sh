#!/bin/bash
# Evidence pass: full GPU suite, bench line, reference arm, launch lists and
# ncu captures (tools/profile_r02.sh) -- everything into gpurun_out/.
cd ${GRAFT_REPO_ROOT:-.}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 2400 python -m pytest tests -q -m gpu -rs --timeout=1200 --durations=60 > gpurun_out/tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/tests.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench rc=$?" >> gpurun_out/bench.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
bash tools/profile_r02.sh > gpurun_out/profile.log 2>&1
ncu --set full --import-source on --clock-control none -f -k regex:k_output -c 1 -o gpurun_out/kout python tools/profile_bfs.py --runs 0 --parents 1 > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/kout.ncu-rep > gpurun_out/kout.txt 2>&1
ncu --set full --import-source on --clock-control none -f -k regex:k_levels8 -c 1 -o gpurun_out/lfb python tools/profile_bfs.py --runs 0 --parents 1 > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/lfb.ncu-rep > gpurun_out/lfb.txt 2>&1
tail -3 gpurun_out/tests.log; tail -c 600 gpurun_out/bench.json; tail -c 300 gpurun_out/bench_ref.json
