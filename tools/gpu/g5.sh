cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -x -rs > gpurun_out/g5_tests.log 2>&1; echo rc=$? >> gpurun_out/g5_tests.log
timeout 900 python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/g5_bench_large.log 2>&1
timeout 600 python bench.py --config medium --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/g5_bench_medium.log 2>&1
