# 4 GPUs, final round-2 code: parity on 4 ranks (peer memory, NCCL; PCG, PC2, CG1, warm starts), the
# 2-GPU test, strong scaling of large (2, 4 GPUs) and medium (4 GPUs), the reference arm at N=4
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
R4="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
R2="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 900 $R4 --master-port 29691 tools/mgpu_check.py > gpurun_out/m6_check_peer4.log 2>&1; echo rc=$? >> gpurun_out/m6_check_peer4.log
POT3D_XFER=0 timeout 900 $R4 --master-port 29692 tools/mgpu_check.py > gpurun_out/m6_check_nccl4.log 2>&1; echo rc=$? >> gpurun_out/m6_check_nccl4.log
timeout 900 python -m pytest -q -m gpu tests/test_multi_gpu.py > gpurun_out/m6_mg_tests.log 2>&1; echo rc=$? >> gpurun_out/m6_mg_tests.log
timeout 900 $R4 --master-port 29693 bench.py --gpus 4 --steps 3 --warmup 3 > gpurun_out/m6_large_n4.log 2>&1
timeout 900 $R2 --master-port 29694 bench.py --gpus 2 --steps 3 --warmup 3 > gpurun_out/m6_large_n2.log 2>&1
timeout 600 $R4 --master-port 29695 bench.py --gpus 4 --config medium --steps 3 --warmup 3 > gpurun_out/m6_medium_n4.log 2>&1
timeout 600 $R4 --master-port 29696 bench.py --impl reference --gpus 4 --steps 2 --warmup 1 > gpurun_out/m6_ref_n4.log 2>&1; echo rc=$? >> gpurun_out/m6_ref_n4.log
