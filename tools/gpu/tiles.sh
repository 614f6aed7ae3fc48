# Tile height variants of the fused passes (tools/build_variants.py tj30 / tj22 / tj30r4) and the
# haloed boxes' L2 promotion: live pass times on large and medium, parity of the 512-thread tiles
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
V=paper_1709_01126_b200/variants
POT3D_LIB=$V/libpot3d_tj30.so timeout 900 python -m pytest -q -m gpu tests/test_gpu_parity.py -k "fused or small or medium" > gpurun_out/t1_tests_tj30.log 2>&1; echo rc=$? >> gpurun_out/t1_tests_tj30.log
for cfg in large medium; do
  for v in default promo128 tj30 tj22 tj30r4 tj30p128; do
    unset POT3D_LIB POT3D_L2PROMO
    case $v in
      promo128) export POT3D_L2PROMO=128;;
      tj30p128) export POT3D_LIB=$V/libpot3d_tj30.so POT3D_L2PROMO=128;;
      default) ;;
      *) export POT3D_LIB=$V/libpot3d_$v.so;;
    esac
    echo "== $v" >> gpurun_out/t1_times_$cfg.log
    timeout 300 python tools/pass_times.py $cfg 200 >> gpurun_out/t1_times_$cfg.log 2>&1
  done
done
unset POT3D_LIB POT3D_L2PROMO
POT3D_LIB=$V/libpot3d_tj30.so timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:"k_pass" -s 6 -c 3 python tools/prof_solve.py large 8 > gpurun_out/t1_ncu_tj30.log 2>&1
