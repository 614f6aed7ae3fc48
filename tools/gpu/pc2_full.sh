# PC2 row-scan sweep with full-tile specialisation: parity tests, checked build, timing variants
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest -q -m gpu tests/test_gpu_parity.py tests/test_loopback.py tests/test_checked_build.py -k "pc2 or spread or fused or checked" > gpurun_out/pc2f_tests.log 2>&1; echo rc=$? >> gpurun_out/pc2f_tests.log
bash tools/gpu/pc2_variants.sh
