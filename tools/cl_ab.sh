for cl in 1 2 4 8; do
  echo "== CL=$cl"
  POT3D_SWEEP_CL=$cl timeout 120 python tools/pc2_dbg2.py 2>&1 | grep -E "rep 2|maxit 10"
  POT3D_SWEEP_CL=$cl timeout 300 python tools/sweep_geom.py 151x64x120 151x301x601 2>&1 | grep tiles
done
POT3D_SWEEP_CL=4 timeout 600 python -m pytest tests -q -m gpu -x -k "pc2 or PC2" 2>&1 | tail -1
