cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_checked_build.py -q --timeout 900 > gpurun_out/g10_checked.log 2>&1; echo rc=$? >> gpurun_out/g10_checked.log
POT3D_LIB=paper_1709_01126_b200/variants/libpot3d_check.so timeout 600 python tools/sanitize_cases.py > gpurun_out/g10_sanitize_cases.log 2>&1; echo rc=$? >> gpurun_out/g10_sanitize_cases.log
