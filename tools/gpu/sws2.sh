# PC2 sweep configuration: tile rows x CTAs per SM, on single problems (medium, large) and a batch
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
V=paper_1709_01126_b200/variants
for v in default sws1 swj16m1; do
  if [ $v = default ]; then unset POT3D_LIB; else export POT3D_LIB=$V/libpot3d_$v.so; fi
  echo "== $v" >> gpurun_out/s2_sweeps.log
  timeout 300 python tools/sweep_geom.py 151x301x601 >> gpurun_out/s2_sweeps.log 2>&1
  timeout 300 python tools/pc2_time.py large 1 >> gpurun_out/s2_sweeps.log 2>&1
  timeout 600 python bench.py --config pc2 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/s2_bench_pc2_$v.log 2>&1
  timeout 600 python bench.py --config batchpc2 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/s2_bench_batchpc2_$v.log 2>&1
done
