mkdir -p gpurun_out
timeout 600 python bench.py --steps 3 --warmup 3 > gpurun_out/n1_bench.log 2>&1; echo "bench rc $?"; tail -1 gpurun_out/n1_bench.log | cut -c1-300
timeout 300 python tools/prof_solve.py medium 30 > gpurun_out/n1_prof_plain.log 2>&1; echo "plain rc $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pass -s 6 -c 2 -o gpurun_out/passes_r01b -f python tools/prof_solve.py medium 30 > gpurun_out/n1_ncu.log 2>&1; echo "ncu rc $?"
