cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/ab; bash tools/p2p_ab.sh adj0 adj2 > gpurun_out/ab/summary.txt 2>&1
