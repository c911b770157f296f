cd $GRAFT_REPO_ROOT
O=gpurun_out/r02_final8; mkdir -p $O
timeout 1500 python -m pytest tests/ -m gpu -q > $O/pytest_gpu_4gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu_4gpu.log
