set -x
mkdir -p gpurun_out
export NCCL_DEBUG=WARN
T="timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29511"
$T tools/mgpu_check.py > gpurun_out/mg4_check.log 2>&1; echo "check rc $?"
tail -8 gpurun_out/mg4_check.log
$T tools/mg_prof.py medium > gpurun_out/mg4_prof.log 2>&1; echo "prof rc $?"; tail -1 gpurun_out/mg4_prof.log
$T bench.py --gpus 4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/mg4_bench.log 2>&1; echo "bench rc $?"; tail -1 gpurun_out/mg4_bench.log | cut -c1-400
$T bench.py --gpus 4 --steps 3 --warmup 3 --no-cpu-baseline --config large > gpurun_out/mg4_bench_large.log 2>&1; echo "bench rc $?"; tail -1 gpurun_out/mg4_bench_large.log | cut -c1-400
$T bench.py --gpus 4 --steps 3 --warmup 3 --no-cpu-baseline --config pc2 > gpurun_out/mg4_bench_pc2.log 2>&1; echo "bench rc $?"; tail -1 gpurun_out/mg4_bench_pc2.log | cut -c1-400
