# PC3 across ranks: loopback tests and the checked build (GPU 0), then tools/mgpu_check.py on 2 GPUs and PC3 medium bench lines
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest -q -m gpu tests/test_pc3.py tests/test_loopback.py tests/test_warm.py tests/test_cg1.py tests/test_checked_build.py > gpurun_out/p3_tests.log 2>&1; echo rc=$? >> gpurun_out/p3_tests.log
R2="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 900 $R2 --master-port 29701 tools/mgpu_check.py > gpurun_out/p3_check_peer2.log 2>&1; echo rc=$? >> gpurun_out/p3_check_peer2.log
POT3D_XFER=0 timeout 900 $R2 --master-port 29702 tools/mgpu_check.py > gpurun_out/p3_check_nccl2.log 2>&1; echo rc=$? >> gpurun_out/p3_check_nccl2.log
timeout 600 $R2 --master-port 29703 bench.py --gpus 2 --config pc3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/p3_bench_pc3_n2.log 2>&1
timeout 900 python -m pytest -q -m gpu tests/test_multi_gpu.py > gpurun_out/p3_mg_tests.log 2>&1; echo rc=$? >> gpurun_out/p3_mg_tests.log
