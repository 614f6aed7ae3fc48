# 4 GPUs: CG1 over peer memory (parity on 2 and 4 ranks, medium / large scaling against PCG and
# CG1 over NCCL) and the edge-shell dispatch (edge-in-A vs the separate kernel) on large
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
R4="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
R2="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 900 $R4 --master-port 29651 tools/mgpu_check.py > gpurun_out/m4_check_peer4.log 2>&1; echo rc=$? >> gpurun_out/m4_check_peer4.log
timeout 900 $R2 --master-port 29652 tools/mgpu_check.py > gpurun_out/m4_check_peer2.log 2>&1; echo rc=$? >> gpurun_out/m4_check_peer2.log
M="bench.py --config medium --steps 3 --warmup 3 --no-cpu-baseline"
timeout 600 $R2 --master-port 29653 $M --gpus 2 > gpurun_out/m4_medium_n2_pcg.log 2>&1
timeout 600 $R2 --master-port 29654 $M --gpus 2 --variant 1 > gpurun_out/m4_medium_n2_cg1.log 2>&1
POT3D_CG1_NCCL=1 timeout 600 $R2 --master-port 29655 $M --gpus 2 --variant 1 > gpurun_out/m4_medium_n2_cg1nccl.log 2>&1
timeout 600 $R4 --master-port 29656 $M --gpus 4 > gpurun_out/m4_medium_n4_pcg.log 2>&1
timeout 600 $R4 --master-port 29657 $M --gpus 4 --variant 1 > gpurun_out/m4_medium_n4_cg1.log 2>&1
POT3D_EDGE_IN_A=0 timeout 600 $R4 --master-port 29658 $M --gpus 4 > gpurun_out/m4_medium_n4_edgek.log 2>&1
L="bench.py --config large --steps 2 --warmup 2 --no-cpu-baseline"
POT3D_EDGE_IN_A=0 timeout 900 $R4 --master-port 29659 $L --gpus 4 > gpurun_out/m4_large_n4_edgek.log 2>&1
timeout 900 $R4 --master-port 29660 $L --gpus 4 --variant 1 > gpurun_out/m4_large_n4_cg1.log 2>&1
POT3D_EDGE_IN_A=0 timeout 900 $R2 --master-port 29661 $L --gpus 2 > gpurun_out/m4_large_n2_edgek.log 2>&1
