cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/ab; bash tools/p2p_ab.sh m20u22 m20u42 m16u82 m24u22 > gpurun_out/ab/summary.txt 2>&1
