# PC2 row-scan sweeps: parity + timing against the run-vectorised sweeps
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "pc2 or medium_fused" --timeout 600 > gpurun_out/g11_pc2tests.log 2>&1; echo rc=$? >> gpurun_out/g11_pc2tests.log
for sw in 0; do
  for b in 1 4; do POT3D_PC2_SWEEP=$sw timeout 300 python tools/pc2_time.py medium $b >> gpurun_out/g11_pc2time.log 2>&1; done
  POT3D_PC2_SWEEP=$sw timeout 300 python tools/pc2_time.py large 1 >> gpurun_out/g11_pc2time.log 2>&1
done
timeout 600 python bench.py --config pc2 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/g11_bench_pc2.log 2>&1
timeout 900 python -m pytest tests/test_loopback.py tests/test_checked_build.py -q --timeout 600 > gpurun_out/g11_loop.log 2>&1; echo rc=$? >> gpurun_out/g11_loop.log
