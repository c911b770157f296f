cd $GRAFT_REPO_ROOT
O=gpurun_out/r02_san; mkdir -p $O
T=$1
timeout 200 python tools/sanitize_case.py > $O/plain_$T.log 2>&1 && \
timeout 1200 /usr/local/cuda/bin/compute-sanitizer --tool $T --print-limit 100 python tools/sanitize_case.py > $O/$T.log 2>&1; echo "rc=$?" >> $O/$T.log
