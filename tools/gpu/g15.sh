cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_pc3.py -q --timeout 600 -x > gpurun_out/g15_pc3.log 2>&1; echo rc=$? >> gpurun_out/g15_pc3.log
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -rs > gpurun_out/g15_tests.log 2>&1; echo rc=$? >> gpurun_out/g15_tests.log
