# CG1 over peer memory: the checked build (every protocol, incl. CG1 loopback)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest -q -m gpu tests/test_checked_build.py > gpurun_out/c9_checked.log 2>&1; echo rc=$? >> gpurun_out/c9_checked.log
