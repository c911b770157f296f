cd $GRAFT_REPO_ROOT
bash tools/profile_round.sh r02_final "r02 final: LET forest, small-leaf P2P variants, subset-cell tensor M2L, far field beside M2L"
