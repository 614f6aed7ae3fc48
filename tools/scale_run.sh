# bench lines at N = 1, 2, 4 on one box (medium, strong scaling) + large at N = 4
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/sc_n1.log 2>&1; echo "n1 rc $?"
for N in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2953$N bench.py --gpus $N > gpurun_out/sc_n$N.log 2>&1; echo "n$N rc $?"
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29539 bench.py --gpus 4 --config large --steps 2 --warmup 3 > gpurun_out/sc_large_n4.log 2>&1; echo "large rc $?"
for f in gpurun_out/sc_n1.log gpurun_out/sc_n2.log gpurun_out/sc_n4.log gpurun_out/sc_large_n4.log; do tail -1 $f | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['n_gpus'], d['config']['workload'][:20], round(d['value'],1), d['unit'], 'e2e', round(d['e2e']['value'],1) if d.get('e2e') else None, 'frac', round(d['roofline']['frac'],3), 'clk', d['clocks']['sm_mhz'], d['clocks']['reasons'])"; done
