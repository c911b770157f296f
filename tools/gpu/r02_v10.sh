cd $GRAFT_REPO_ROOT
O=gpurun_out/r02_v10; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q -s -k "not mgpu" > $O/gpu_tests.log 2>&1; echo "tests rc=$?" >> $O/gpu_tests.log
timeout 600 python tools/p2p_sweep.py --reps 5 > $O/p2p.log 2>&1
