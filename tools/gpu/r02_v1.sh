set -x
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02_v1; mkdir -p $O
nvidia-smi --query-gpu=name,memory.total --format=csv > $O/gpu.txt; nproc >> $O/gpu.txt; free -g >> $O/gpu.txt
timeout 1500 python -m pytest tests -m gpu -x -q -s -k "not mgpu" > $O/gpu_tests.log 2>&1; echo "tests rc=$?" >> $O/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
timeout 600 python bench.py --workload advected --no-cpu-baseline --no-e2e > $O/bench_advected.json 2> $O/bench_advected.err
timeout 600 python bench.py --workload jitter --no-cpu-baseline --no-e2e > $O/bench_jitter.json 2> $O/bench_jitter.err
