# Thread-block clusters of neighbouring tiles for the fused passes (POT3D_CLUSTER=JxK):
# parity with clusters, live pass times, ncu DRAM bytes / L2 hit rate of pass A
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for cl in 2x1 2x2; do
  POT3D_CLUSTER=$cl timeout 600 python -m pytest -q -m gpu tests/test_gpu_parity.py -k "fused or small" > gpurun_out/c1_tests_$cl.log 2>&1; echo rc=$? >> gpurun_out/c1_tests_$cl.log
done
for cfg in large medium; do
  for cl in 1x1 2x1 4x1 8x1 2x2 1x2 4x2; do
    echo "== $cl" >> gpurun_out/c1_times_$cfg.log
    POT3D_CLUSTER=$cl timeout 300 python tools/pass_times.py $cfg 200 >> gpurun_out/c1_times_$cfg.log 2>&1
  done
done
for cl in 1x1 2x1 4x1 2x2; do
  POT3D_CLUSTER=$cl timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:"k_pass_a|k_pass_b_pc1" -s 6 -c 3 python tools/prof_solve.py large 8 > gpurun_out/c1_ncu_$cl.log 2>&1
done
