cd $GRAFT_REPO_ROOT
bash tools/profile_round.sh r02_prof2 "r02 v9: small-leaf variants, P2P list grouped by target"
