# 4 GPUs: CG1 over peer memory with parity-alternating mailbox slots; the adaptive edge-shell dispatch
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
R4="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
R2="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 900 $R4 --master-port 29671 tools/mgpu_check.py > gpurun_out/m5_check_peer4.log 2>&1; echo rc=$? >> gpurun_out/m5_check_peer4.log
M="bench.py --config medium --steps 3 --warmup 3 --no-cpu-baseline"
timeout 600 $R4 --master-port 29672 $M --gpus 4 --variant 1 > gpurun_out/m5_medium_n4_cg1.log 2>&1
timeout 600 $R2 --master-port 29673 $M --gpus 2 --variant 1 > gpurun_out/m5_medium_n2_cg1.log 2>&1
timeout 600 $R4 --master-port 29674 $M --gpus 4 > gpurun_out/m5_medium_n4_pcg.log 2>&1
L="bench.py --config large --steps 3 --warmup 3"
timeout 900 $R4 --master-port 29675 $L --gpus 4 > gpurun_out/m5_large_n4.log 2>&1
timeout 900 $R2 --master-port 29676 $L --gpus 2 > gpurun_out/m5_large_n2.log 2>&1
timeout 900 $R4 --master-port 29677 $L --gpus 4 --variant 1 > gpurun_out/m5_large_n4_cg1.log 2>&1
timeout 900 python -m pytest -q -m gpu tests/test_multi_gpu.py > gpurun_out/m5_mg_tests.log 2>&1; echo rc=$? >> gpurun_out/m5_mg_tests.log
