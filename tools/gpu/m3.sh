# 4 GPUs, final code: parity on 4 and 2 ranks (peer memory and NCCL, incl. CG1), strong scaling of large and medium
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
R4="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
R2="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 900 $R4 --master-port 29631 tools/mgpu_check.py > gpurun_out/m3_check_peer.log 2>&1; echo rc=$? >> gpurun_out/m3_check_peer.log
POT3D_XFER=0 timeout 900 $R4 --master-port 29632 tools/mgpu_check.py > gpurun_out/m3_check_nccl.log 2>&1; echo rc=$? >> gpurun_out/m3_check_nccl.log
timeout 900 python -m pytest -q -m gpu tests/test_multi_gpu.py > gpurun_out/m3_mg_tests.log 2>&1; echo rc=$? >> gpurun_out/m3_mg_tests.log
timeout 900 $R4 --master-port 29633 bench.py --gpus 4 --steps 3 --warmup 3 > gpurun_out/m3_bench_large_n4.log 2>&1
timeout 900 $R2 --master-port 29634 bench.py --gpus 2 --steps 3 --warmup 3 > gpurun_out/m3_bench_large_n2.log 2>&1
timeout 600 $R4 --master-port 29635 bench.py --gpus 4 --config medium --steps 3 --warmup 3 > gpurun_out/m3_bench_medium_n4.log 2>&1
timeout 600 $R4 --master-port 29636 bench.py --gpus 4 --config medium --steps 3 --warmup 3 --variant 1 > gpurun_out/m3_bench_medium_n4_cg1.log 2>&1
timeout 600 $R4 --master-port 29637 bench.py --gpus 4 --config pc2 --steps 3 --warmup 3 > gpurun_out/m3_bench_pc2_n4.log 2>&1
timeout 900 $R4 --master-port 29638 bench.py --impl reference --gpus 4 --steps 2 --warmup 1 > gpurun_out/m3_bench_ref_n4.log 2>&1; echo rc=$? >> gpurun_out/m3_bench_ref_n4.log
