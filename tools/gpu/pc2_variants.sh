# PC2 row-scan sweeps: tile rows (POT3D_SWJ) and prefetch depth (POT3D_SPD) variants
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in default swj4 swj16 spd1; do
  if [ $v = default ]; then unset POT3D_LIB; else export POT3D_LIB=paper_1709_01126_b200/variants/libpot3d_$v.so; fi
  echo "== $v" >> gpurun_out/pc2_variants.log
  timeout 300 python tools/sweep_geom.py 151x8x120 151x64x120 151x301x601 >> gpurun_out/pc2_variants.log 2>&1
  timeout 300 python tools/pc2_time.py large 1 >> gpurun_out/pc2_variants.log 2>&1
done
