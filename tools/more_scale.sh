T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 $T --nproc-per-node 2 --master-port 29651 bench.py --gpus 2 --config large --steps 1 --warmup 3 --no-e2e > gpurun_out/ms_large_n2.log 2>&1; echo "large2 rc $?"
timeout 900 $T --nproc-per-node 4 --master-port 29652 bench.py --gpus 4 --config large --steps 1 --warmup 3 --no-e2e > gpurun_out/ms_large_n4.log 2>&1; echo "large4 rc $?"
timeout 900 $T --nproc-per-node 2 --master-port 29653 bench.py --gpus 2 --config pc2 --steps 2 --warmup 3 --no-e2e > gpurun_out/ms_pc2_n2.log 2>&1; echo "pc2_2 rc $?"
timeout 900 $T --nproc-per-node 4 --master-port 29654 bench.py --gpus 4 --config pc2 --steps 2 --warmup 3 --no-e2e > gpurun_out/ms_pc2_n4.log 2>&1; echo "pc2_4 rc $?"
timeout 900 $T --nproc-per-node 4 --master-port 29655 bench.py --gpus 4 --config weak --steps 2 --warmup 3 > gpurun_out/ms_weak_n4.log 2>&1; echo "weak4 rc $?"
for f in gpurun_out/ms_*.log; do tail -1 $f | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$f', d['n_gpus'], d['config']['workload'][:12], round(d['value'],1), 'tts', round(d['time_to_solve_s'],3), 'iters', d['config']['iters_per_step'][0])"; done
