cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in spd3 spd4 spd6; do
  POT3D_LIB=paper_1709_01126_b200/variants/libpot3d_$v.so timeout 300 python tools/sweep_geom.py 151x8x120 151x64x120 151x301x601 > gpurun_out/g14_geom_$v.log 2>&1
done
timeout 900 python -m pytest tests/test_gpu_parity.py -q -s -k "spread" --timeout 600 > gpurun_out/g14_spread.log 2>&1
