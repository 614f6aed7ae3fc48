# 4 GPUs: PC3 with peer-memory d halos (parity on 4 ranks, medium / large lines); the checked build's new cases (GPU 0)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
R4="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
timeout 900 python -m pytest -q -m gpu tests/test_checked_build.py > gpurun_out/m9_checked.log 2>&1; echo rc=$? >> gpurun_out/m9_checked.log
timeout 900 $R4 --master-port 29721 tools/mgpu_check.py > gpurun_out/m9_check_peer4.log 2>&1; echo rc=$? >> gpurun_out/m9_check_peer4.log
timeout 600 $R4 --master-port 29722 bench.py --gpus 4 --config pc3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/m9_pc3_n4.log 2>&1
timeout 600 $R4 --master-port 29723 bench.py --gpus 4 --config pc3large --steps 2 --warmup 2 --no-cpu-baseline > gpurun_out/m9_pc3large_n4.log 2>&1
