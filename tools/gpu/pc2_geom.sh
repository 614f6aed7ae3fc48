cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python tools/sweep_geom.py 151x8x120 151x16x120 151x64x120 151x8x600 151x301x120 151x64x600 151x301x601 > gpurun_out/g13_geom_scan.log 2>&1
POT3D_PC2_SWEEP=4 timeout 600 python tools/sweep_geom.py 151x8x120 151x64x120 151x301x601 > gpurun_out/g13_geom_s4.log 2>&1
