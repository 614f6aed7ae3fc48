# the round's last code on one GPU: the GPU suite, smoke, the default bench line and the reference arm
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 -rs > gpurun_out/f6_tests.log 2>&1; echo "rc=$?" >> gpurun_out/f6_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f6_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/f6_smoke.log
timeout 1500 python bench.py > gpurun_out/f6_bench_n1.log 2>&1; echo "rc=$?" >> gpurun_out/f6_bench_n1.log
timeout 600 python bench.py --impl reference > gpurun_out/f6_bench_ref.log 2>&1; echo "rc=$?" >> gpurun_out/f6_bench_ref.log
