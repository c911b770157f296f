cd $GRAFT_REPO_ROOT
O=gpurun_out/r02_poison; mkdir -p $O
V=paper_1106_5273_b200/build/variants
timeout 1200 python -m pytest tests/test_gpu_poison.py -x -q > $O/poison.log 2>&1; echo "rc=$?" >> $O/poison.log
for v in bug_lc bug_oob; do
  FMM_LIB=$V/$v/libfmm_b200.so timeout 600 python -m pytest tests/test_gpu_poison.py -x -q > $O/poison_$v.log 2>&1; echo "rc=$?" >> $O/poison_$v.log
  FMM_LIB=$V/$v/libfmm_b200.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py -q > $O/parity_$v.log 2>&1; echo "rc=$?" >> $O/parity_$v.log
done
