# Round evidence on one GPU: tests, bench line, ncu launch list, ncu --set full of the passes
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/pr_tests.log 2>&1; echo "tests rc $?"; tail -2 gpurun_out/pr_tests.log
timeout 900 python bench.py > gpurun_out/pr_bench.log 2>&1; echo "bench rc $?"; tail -1 gpurun_out/pr_bench.log | cut -c1-200
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 30000 -c 400 --csv --log-file gpurun_out/pr_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/pr_ncu_launch.log 2>&1; echo "ncu launches rc $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pass -s 6 -c 2 -o gpurun_out/pr_passes -f python tools/prof_solve.py medium 30 > gpurun_out/pr_ncu_full.log 2>&1; echo "ncu full rc $?"
