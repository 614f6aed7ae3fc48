# Multi-RHS batches: parity tests, PC2 tests (prefetch depth 1), bench lines (batch, batchsmall, small)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest -q -m gpu tests/test_batch.py -x > gpurun_out/b1_batch_tests.log 2>&1; echo rc=$? >> gpurun_out/b1_batch_tests.log
timeout 900 python -m pytest -q -m gpu tests/test_gpu_parity.py tests/test_loopback.py -k "pc2 or spread" > gpurun_out/b1_pc2_tests.log 2>&1; echo rc=$? >> gpurun_out/b1_pc2_tests.log
timeout 600 python bench.py --config batch --steps 3 --warmup 3 > gpurun_out/b1_bench_batch.log 2>&1
timeout 600 python bench.py --config medium --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/b1_bench_medium.log 2>&1
timeout 300 python bench.py --config batchsmall --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/b1_bench_batchsmall.log 2>&1
timeout 300 python bench.py --config small --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/b1_bench_small.log 2>&1
timeout 300 python bench.py --config pc2 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/b1_bench_pc2.log 2>&1
