# 4 GPUs, last code: parity on 4 ranks (peer memory / NCCL: PCG PC1/PC2, CG1, PC3, warm starts), PC3 and PCG medium lines
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
R4="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
timeout 900 $R4 --master-port 29711 tools/mgpu_check.py > gpurun_out/m8_check_peer4.log 2>&1; echo rc=$? >> gpurun_out/m8_check_peer4.log
POT3D_XFER=0 timeout 900 $R4 --master-port 29712 tools/mgpu_check.py > gpurun_out/m8_check_nccl4.log 2>&1; echo rc=$? >> gpurun_out/m8_check_nccl4.log
timeout 600 $R4 --master-port 29713 bench.py --gpus 4 --config pc3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/m8_pc3_n4.log 2>&1
timeout 600 $R4 --master-port 29714 bench.py --gpus 4 --config pc3large --steps 2 --warmup 2 --no-cpu-baseline > gpurun_out/m8_pc3large_n4.log 2>&1
