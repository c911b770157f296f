cd $GRAFT_REPO_ROOT
O=gpurun_out/r02_m4; mkdir -p $O
timeout 900 python -m pytest tests/test_mgpu.py -q -s -k "edge or (orb_partition and 3)" > $O/mgpu_edge.log 2>&1; echo "rc=$?" >> $O/mgpu_edge.log
