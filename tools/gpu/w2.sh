# warm starts across ranks: loopback tests (GPU 0) and tools/mgpu_check.py on 2 GPUs (peer memory and NCCL)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest -q -m gpu tests/test_warm.py tests/test_cg1.py tests/test_loopback.py > gpurun_out/w2_tests.log 2>&1; echo rc=$? >> gpurun_out/w2_tests.log
R2="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 900 $R2 --master-port 29681 tools/mgpu_check.py > gpurun_out/w2_check_peer2.log 2>&1; echo rc=$? >> gpurun_out/w2_check_peer2.log
POT3D_XFER=0 timeout 900 $R2 --master-port 29682 tools/mgpu_check.py > gpurun_out/w2_check_nccl2.log 2>&1; echo rc=$? >> gpurun_out/w2_check_nccl2.log
