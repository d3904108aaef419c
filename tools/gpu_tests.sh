cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gputest_r02e.log 2>&1; echo "tests rc=$?"; tail -4 gpurun_out/gputest_r02e.log
for s in 81 82; do timeout 900 python tools/stress_parity.py $s 150 > gpurun_out/stress_r02e_$s.log 2>&1; echo "stress $s rc=$?"; tail -2 gpurun_out/stress_r02e_$s.log; done
