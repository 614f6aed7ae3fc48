# PC3 init kernel rewritten by rows: parity (PC3 tests, loopback, checked build) and the ncu time, medium PC3 lines
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest -q -m gpu tests/test_pc3.py tests/test_batch.py tests/test_checked_build.py tests/test_warm.py > gpurun_out/pi_tests.log 2>&1; echo rc=$? >> gpurun_out/pi_tests.log
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_poly_init" -s 2 -c 2 python tools/prof_solve.py medium 4 3 > gpurun_out/pi_ncu.log 2>&1
timeout 600 python bench.py --config pc3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/pi_bench_pc3.log 2>&1
timeout 600 python bench.py --config pc3 --poly 8,1000 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/pi_bench_pc3_m8.log 2>&1
