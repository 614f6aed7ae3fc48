# weak scaling: 554 G x 601 x 1201 cells, fixed 300 iterations per step
timeout 900 python bench.py --config weak --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/wk_n1.log 2>&1; echo "n1 rc $?"
for N in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2955$N bench.py --gpus $N --config weak --steps 2 --warmup 3 > gpurun_out/wk_n$N.log 2>&1; echo "n$N rc $?"
done
for N in 1 2 4; do tail -1 gpurun_out/wk_n$N.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['n_gpus'], d['config']['cells'], round(d['value'],1), d['unit'], 'ms/step', round(d['ms_per_step'],1), 'frac', round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])"; done
