cd $GRAFT_REPO_ROOT
O=gpurun_out/r02_sweep3; mkdir -p $O
V=paper_1106_5273_b200/build/variants
for v in default u6n2 u7n3 u6n4 default; do
  if [ $v = default ]; then L=""; else L="FMM_LIB=$V/$v/libfmm_b200.so"; fi
  env $L timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e >> $O/b_$v.json 2>> $O/b_$v.err
done
