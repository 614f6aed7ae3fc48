# 4 GPUs: parity on 4 ranks (peer memory and NCCL, incl. CG1), strong scaling of large and medium, PC2
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
timeout 900 $R --master-port 29621 tools/mgpu_check.py > gpurun_out/m2_check_peer.log 2>&1; echo rc=$? >> gpurun_out/m2_check_peer.log
POT3D_XFER=0 timeout 900 $R --master-port 29622 tools/mgpu_check.py > gpurun_out/m2_check_nccl.log 2>&1; echo rc=$? >> gpurun_out/m2_check_nccl.log
timeout 900 $R --master-port 29623 bench.py --gpus 4 --steps 3 --warmup 2 > gpurun_out/m2_bench_large_n4.log 2>&1
timeout 600 $R --master-port 29624 bench.py --gpus 4 --config medium --steps 3 --warmup 2 > gpurun_out/m2_bench_medium_n4.log 2>&1
timeout 600 $R --master-port 29625 bench.py --gpus 4 --config pc2 --steps 3 --warmup 2 > gpurun_out/m2_bench_pc2_n4.log 2>&1
timeout 600 $R --master-port 29626 bench.py --gpus 4 --config medium --steps 3 --warmup 2 --variant 1 > gpurun_out/m2_bench_medium_n4_cg1.log 2>&1
