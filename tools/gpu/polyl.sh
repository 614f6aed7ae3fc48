# PC3 with 8 Chebyshev steps on large: 1 and 4 GPUs
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
R4="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
timeout 900 $R4 --master-port 29741 bench.py --gpus 4 --config pc3large --poly 8,100 --steps 2 --warmup 2 --no-cpu-baseline > gpurun_out/pl_n4_m8.log 2>&1
timeout 1200 python bench.py --config pc3large --poly 8,100 --steps 2 --warmup 2 --no-cpu-baseline > gpurun_out/pl_n1_m8.log 2>&1
