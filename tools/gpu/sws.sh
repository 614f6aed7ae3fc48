# Row-scan sweeps at two CTAs per SM (POT3D_SWS_MINB=2, default) vs one (sws1), tile-height variants
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest -q -m gpu tests/test_gpu_parity.py tests/test_loopback.py > gpurun_out/s1_pc2_tests.log 2>&1; echo rc=$? >> gpurun_out/s1_pc2_tests.log
for cfg in large medium; do timeout 300 python tools/pass_times.py $cfg 200 >> gpurun_out/s1_pass_times.log 2>&1; done
timeout 900 python -m pytest -q -m gpu tests/test_batch.py tests/test_pc3.py > gpurun_out/s1_batch_tests.log 2>&1; echo rc=$? >> gpurun_out/s1_batch_tests.log
V=paper_1709_01126_b200/variants
for v in default sws1 swj16m1 swj4; do
  if [ $v = default ]; then unset POT3D_LIB; else export POT3D_LIB=$V/libpot3d_$v.so; fi
  echo "== $v" >> gpurun_out/s1_sweeps.log
  timeout 300 python tools/sweep_geom.py 151x8x120 151x301x601 >> gpurun_out/s1_sweeps.log 2>&1
  timeout 300 python tools/pc2_time.py large 1 >> gpurun_out/s1_sweeps.log 2>&1
done
unset POT3D_LIB
timeout 600 python bench.py --config pc2 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/s1_bench_pc2.log 2>&1
timeout 600 python bench.py --config batchpc2 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/s1_bench_batchpc2.log 2>&1
timeout 600 python bench.py --config batchpc3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/s1_bench_batchpc3.log 2>&1
timeout 600 python bench.py --config pc3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/s1_bench_pc3.log 2>&1
