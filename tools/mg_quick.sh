# multi-GPU: parity check + bench + thin-slab latency (N GPUs)
N=${1:-4}
T="timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29517"
$T tools/mgpu_check.py > gpurun_out/mgq_check.log 2>&1; echo "check rc $?"; grep -c " OK " gpurun_out/mgq_check.log; grep FAIL gpurun_out/mgq_check.log
$T bench.py --gpus $N --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | cut -c1-160
$T tools/lat.py 76x301x601 400 2>&1 | grep us/iter
$T tools/lat.py medium 400 2>&1 | grep us/iter
