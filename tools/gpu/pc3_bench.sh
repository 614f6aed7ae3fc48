cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -s -k "golden or spread" --timeout 600 > gpurun_out/g16_golden.log 2>&1; echo rc=$? >> gpurun_out/g16_golden.log
timeout 900 python bench.py --config pc3 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/g16_bench_pc3.log 2>&1
timeout 1200 python bench.py --config pc3large --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/g16_bench_pc3large.log 2>&1
timeout 1200 python bench.py --config pc2 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/g16_bench_pc2.log 2>&1
