# round evidence: GPU tests, smoke, bench N=1 (+ ncu launch list, ncu full), N=2/4 bench lines
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu > gpurun_out/fe_tests.log 2>&1; echo "tests rc $?"; tail -1 gpurun_out/fe_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fe_smoke.log 2>&1; echo "smoke rc $?"; tail -1 gpurun_out/fe_smoke.log
timeout 900 python bench.py > gpurun_out/fe_n1.log 2>&1; echo "bench rc $?"
for N in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2959$N bench.py --gpus $N > gpurun_out/fe_n$N.log 2>&1; echo "n$N rc $?"
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 30000 -c 400 --csv --log-file gpurun_out/fe_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/fe_ncu_launch.log 2>&1; echo "ncu launches rc $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pass -s 6 -c 2 -o gpurun_out/fe_passes -f python tools/prof_solve.py medium 30 > gpurun_out/fe_ncu_full.log 2>&1; echo "ncu full rc $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sweep4 -s 2 -c 2 -o gpurun_out/fe_sweeps -f python tools/prof_solve.py medium 6 2 > gpurun_out/fe_ncu_sweep.log 2>&1; echo "ncu sweep rc $?"
for f in gpurun_out/fe_n1.log gpurun_out/fe_n2.log gpurun_out/fe_n4.log; do tail -1 $f | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['n_gpus'], round(d['value'],1), 'e2e', round(d['e2e']['value'],1), 'frac', round(d['roofline']['frac'],3), d['clocks']['sm_mhz'], d['clocks']['reasons'])"; done
