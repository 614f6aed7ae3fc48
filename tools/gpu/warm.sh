# Multi-RHS batches and warm starts: parity tests, then the batch bench lines
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest -q -m gpu tests/test_batch.py tests/test_warm.py > gpurun_out/w1_tests.log 2>&1; echo rc=$? >> gpurun_out/w1_tests.log
timeout 600 python -m pytest -q -m gpu tests/test_gpu_parity.py -x > gpurun_out/w1_parity.log 2>&1; echo rc=$? >> gpurun_out/w1_parity.log
