# 2 GPUs: multi-GPU parity (peer memory, NCCL, CG1), bench N=2 large / medium, standard and CG1
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi topo -m > gpurun_out/m1_topo.txt 2>&1
timeout 1200 python -m pytest tests/test_multi_gpu.py -q -s --timeout 1100 > gpurun_out/m1_tests.log 2>&1; echo rc=$? >> gpurun_out/m1_tests.log
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 900 $R --master-port 29611 bench.py --gpus 2 --steps 2 --warmup 1 > gpurun_out/m1_bench_large_n2.log 2>&1
timeout 600 $R --master-port 29612 bench.py --gpus 2 --config medium --steps 3 --warmup 2 > gpurun_out/m1_bench_medium_n2.log 2>&1
timeout 600 $R --master-port 29613 bench.py --gpus 2 --config medium --steps 3 --warmup 2 --variant 1 > gpurun_out/m1_bench_medium_n2_cg1.log 2>&1
timeout 900 $R --master-port 29614 bench.py --gpus 2 --steps 2 --warmup 1 --variant 1 > gpurun_out/m1_bench_large_n2_cg1.log 2>&1
