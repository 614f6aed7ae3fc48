# loopback + full GPU tests
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_loopback.py -q -x --timeout 300 > gpurun_out/g3_loop.log 2>&1; echo rc=$? >> gpurun_out/g3_loop.log
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/g3_tests.log 2>&1; echo rc=$? >> gpurun_out/g3_tests.log
