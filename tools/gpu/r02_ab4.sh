cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/ab; bash tools/p2p_ab.sh nocls > gpurun_out/ab/summary4.txt 2>&1
