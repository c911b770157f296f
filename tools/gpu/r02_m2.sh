cd $GRAFT_REPO_ROOT
O=gpurun_out/r02_m2; mkdir -p $O
nvidia-smi -L > $O/gpus.txt
timeout 900 python -m pytest tests/test_mgpu.py -q -s > $O/mgpu_tests.log 2>&1; echo "rc=$?" >> $O/mgpu_tests.log
timeout 900 python -m pytest tests -m gpu -q -s -k "not mgpu and not c4" > $O/gpu_tests.log 2>&1; echo "rc=$?" >> $O/gpu_tests.log
