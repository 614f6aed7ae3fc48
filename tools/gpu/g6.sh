cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_cg1.py -q --timeout 300 -rs > gpurun_out/g6_cg1.log 2>&1; echo rc=$? >> gpurun_out/g6_cg1.log
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -rs > gpurun_out/g6_tests.log 2>&1; echo rc=$? >> gpurun_out/g6_tests.log
