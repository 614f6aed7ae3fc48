# PC2 batches: parity, then bench lines (batchpc2 vs pc2)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest -q -m gpu tests/test_batch.py tests/test_warm.py > gpurun_out/p2_tests.log 2>&1; echo rc=$? >> gpurun_out/p2_tests.log
timeout 900 python -m pytest -q -m gpu tests/test_gpu_parity.py tests/test_loopback.py -k "pc2 or spread" > gpurun_out/p2_pc2_tests.log 2>&1; echo rc=$? >> gpurun_out/p2_pc2_tests.log
timeout 600 python bench.py --config batchpc2 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/p2_bench_batchpc2.log 2>&1
timeout 600 python bench.py --config pc2 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/p2_bench_pc2.log 2>&1
