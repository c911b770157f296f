cd $GRAFT_REPO_ROOT
O=gpurun_out/r02_let; mkdir -p $O
for P in 3 4; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $P --master-addr 127.0.0.1 --master-port 2961$P tools/let_compare.py > $O/let_p$P.log 2>&1
done
