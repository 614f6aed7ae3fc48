# L2 promotion of the TMA boxes (POT3D_L2PROMO): live pass times and ncu DRAM bytes
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for cfg in large medium; do
  for pr in 128 0 64 256; do
    echo "== $pr" >> gpurun_out/l2_times_$cfg.log
    POT3D_L2PROMO=$pr timeout 300 python tools/pass_times.py $cfg 200 >> gpurun_out/l2_times_$cfg.log 2>&1
  done
done
for pr in 0 64 256; do
  POT3D_L2PROMO=$pr timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:"k_pass" -s 6 -c 3 python tools/prof_solve.py large 8 > gpurun_out/l2_ncu_$pr.log 2>&1
done
