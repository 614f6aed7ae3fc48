cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -rs > gpurun_out/g4_tests.log 2>&1; echo rc=$? >> gpurun_out/g4_tests.log
