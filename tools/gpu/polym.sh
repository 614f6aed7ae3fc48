# PC3 Chebyshev steps m (2 .. 8) on medium: time to solution on 1 and 4 GPUs
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
R4="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
port=29730
for m in 2 3 6 8; do
  timeout 600 python bench.py --config pc3 --poly $m,100 --steps 2 --warmup 2 --no-cpu-baseline > gpurun_out/pm_n1_m$m.log 2>&1
  port=$((port+1))
  timeout 600 $R4 --master-port $port bench.py --gpus 4 --config pc3 --poly $m,100 --steps 2 --warmup 2 --no-cpu-baseline > gpurun_out/pm_n4_m$m.log 2>&1
done
