cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/g1_smi.txt
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/g1_tests.log 2>&1; echo rc=$? >> gpurun_out/g1_tests.log
timeout 600 python tools/parity_probe.py > gpurun_out/g1_probe.log 2>&1
timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/g1_bench_medium.log 2>&1
timeout 600 python bench.py --config large --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/g1_bench_large.log 2>&1
