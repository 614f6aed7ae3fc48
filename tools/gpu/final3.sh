# final round-2 evidence on one GPU: tests, smoke, bench (driver command shape), reference arm,
# launch list, ncu --set full of the passes (large, medium) and the PC2 sweeps (medium)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 -rs > gpurun_out/f3_tests.log 2>&1; echo "rc=$?" >> gpurun_out/f3_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f3_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/f3_smoke.log
timeout 1500 python bench.py --gpus 1 --steps 5 --warmup 3 > gpurun_out/f3_bench_n1.log 2>&1; echo "rc=$?" >> gpurun_out/f3_bench_n1.log
timeout 600 python bench.py --impl reference --gpus 1 --steps 5 --warmup 3 > gpurun_out/f3_bench_ref.log 2>&1; echo "rc=$?" >> gpurun_out/f3_bench_ref.log
timeout 600 python bench.py --config medium --steps 3 --warmup 3 > gpurun_out/f3_bench_medium.log 2>&1; echo "rc=$?" >> gpurun_out/f3_bench_medium.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/f3_launches.csv python tools/prof_solve.py large 200 > gpurun_out/f3_ncu_launch.log 2>&1; echo "rc=$?" >> gpurun_out/f3_ncu_launch.log
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_pass" -s 6 -c 4 -o gpurun_out/f3_passes_large -f python tools/prof_solve.py large 10 > gpurun_out/f3_ncu_full.log 2>&1; echo "rc=$?" >> gpurun_out/f3_ncu_full.log
python tools/ncu_summary.py gpurun_out/f3_passes_large.ncu-rep > gpurun_out/f3_ncu_summary.txt 2>&1
timeout 900 ncu --set full --clock-control none -k regex:"k_pass" -s 6 -c 4 -o gpurun_out/f3_passes_medium -f python tools/prof_solve.py medium 10 > gpurun_out/f3_ncu_full_medium.log 2>&1
python tools/ncu_summary.py gpurun_out/f3_passes_medium.ncu-rep > gpurun_out/f3_ncu_summary_medium.txt 2>&1
timeout 900 ncu --set full --clock-control none -k regex:"k_sweepS|k_pass" -s 4 -c 5 -o gpurun_out/f3_pc2_medium -f python tools/prof_solve.py medium 4 2 > gpurun_out/f3_ncu_full_pc2.log 2>&1
python tools/ncu_summary.py gpurun_out/f3_pc2_medium.ncu-rep > gpurun_out/f3_ncu_summary_pc2.txt 2>&1
timeout 600 python bench.py --config pc2 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/f3_bench_pc2.log 2>&1
timeout 600 python bench.py --config batch --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/f3_bench_batch.log 2>&1
timeout 600 python bench.py --config batchpc2 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/f3_bench_batchpc2.log 2>&1
