cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gputest_r02b.log 2>&1; echo "tests rc=$?"; tail -5 gpurun_out/gputest_r02b.log
LIBS="abl/b512.so paper_2605_10433_b200/libqsg.so" bash tools/ab3.sh 254 bp4 0.02,0.06,0.08,0.1 > gpurun_out/ab3.log 2>&1
LIBS="abl/b512.so paper_2605_10433_b200/libqsg.so" bash tools/ab3.sh 1022,rgb127w8 bp4 0.04,0.08 >> gpurun_out/ab3.log 2>&1
python tools/ab_table.py gpurun_out/ab3.log
TAG=bp4_r02b VAR=bp4 P=0.1 STEPS=ncu bash tools/gpu_session.sh
