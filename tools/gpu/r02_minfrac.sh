cd $GRAFT_REPO_ROOT
O=gpurun_out/r02_minfrac; mkdir -p $O
V=paper_1106_5273_b200/build/variants
for v in default mf25 mf33 mf55; do
  if [ $v = default ]; then L=""; else L="FMM_LIB=$V/$v/libfmm_b200.so"; fi
  env $L timeout 300 python bench.py --workload jitter --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $O/jit_$v.json 2> $O/jit_$v.err
  env $L timeout 300 python bench.py --workload advected --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $O/adv_$v.json 2> $O/adv_$v.err
done
