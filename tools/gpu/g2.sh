# round 2: GPU tests, parity probe, bench on large (default) and medium, ncu on the passes (large)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/g2_tests.log 2>&1; echo rc=$? >> gpurun_out/g2_tests.log
timeout 600 python tools/parity_probe.py > gpurun_out/g2_probe.log 2>&1
timeout 900 python bench.py --steps 2 --warmup 1 > gpurun_out/g2_bench_large.log 2>&1
timeout 600 python bench.py --config medium --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/g2_bench_medium.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pass -s 6 -c 4 -o gpurun_out/g2_passes_large -f python tools/prof_solve.py large 12 > gpurun_out/g2_ncu.log 2>&1
python tools/ncu_summary.py gpurun_out/g2_passes_large.ncu-rep > gpurun_out/g2_ncu_summary.txt 2>&1
