set -x
mkdir -p gpurun_out
export NCCL_DEBUG=WARN
T="timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511"
$T tools/mgpu_check.py > gpurun_out/mg2_check.log 2>&1; echo "check rc $?"
tail -12 gpurun_out/mg2_check.log
$T tools/mg_prof.py medium > gpurun_out/mg2_prof.log 2>&1; echo "prof rc $?"; tail -3 gpurun_out/mg2_prof.log
POT3D_XFER=0 $T tools/mg_prof.py medium > gpurun_out/mg2_prof_nccl.log 2>&1; tail -2 gpurun_out/mg2_prof_nccl.log
$T bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/mg2_bench.log 2>&1; echo "bench rc $?"; tail -2 gpurun_out/mg2_bench.log
POT3D_XFER=0 $T bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/mg2_bench_nccl.log 2>&1; tail -1 gpurun_out/mg2_bench_nccl.log
