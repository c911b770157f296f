cd $GRAFT_REPO_ROOT
O=gpurun_out/r02_chunk; mkdir -p $O
V=paper_1106_5273_b200/build/variants
for v in default c48 c64; do
  if [ $v = default ]; then L=""; else L="FMM_LIB=$V/$v/libfmm_b200.so"; fi
  env $L timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $O/b_$v.json 2> $O/b_$v.err
  env $L timeout 600 python -m pytest tests/test_gpu_m2l_tc.py tests/test_gpu_parity.py -x -q -s > $O/t_$v.log 2>&1; echo "rc=$?" >> $O/t_$v.log
done
