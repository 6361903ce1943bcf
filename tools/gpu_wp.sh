cd $GRAFT_REPO_ROOT
SW_ROOTS=16 timeout 900 python tools/expand_sweep.py libbflybfs_wp0.so libbflybfs.so libbflybfs_wp0.so libbflybfs.so > gpurun_out/sweep.log 2>&1
grep "parents=True" gpurun_out/sweep.log
timeout 1500 python -m pytest tests -q -x -m gpu --timeout=900 -k "parents or golden or config or parity or dist or readout or acceptance_sweep or deep or tiny" > gpurun_out/tp.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/tp.log
