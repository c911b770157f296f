cd $GRAFT_REPO_ROOT
bash tools/profile_round.sh r02_prof1 "r02: adjacency 32-source tiles, rho>=4.6 singular branch"
