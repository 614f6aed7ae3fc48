# full GPU suite and the PC2 / batch bench lines after the sweep-tile and shared-face changes
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 -rs > gpurun_out/v3_tests.log 2>&1; echo "rc=$?" >> gpurun_out/v3_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/v3_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/v3_smoke.log
timeout 600 python bench.py --config pc2 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/v3_bench_pc2.log 2>&1
timeout 600 python bench.py --config batchpc2 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/v3_bench_batchpc2.log 2>&1
timeout 900 python bench.py --config large --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/v3_bench_large.log 2>&1
