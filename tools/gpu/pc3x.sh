# PC3: interval ratio sweep at 8 steps (medium, 1 GPU) and ncu --set full of the Chebyshev kernels (traffic.json "pc3")
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for r in 30 300 1000 3000; do
  timeout 600 python bench.py --config pc3 --poly 8,$r --steps 2 --warmup 2 --no-cpu-baseline > gpurun_out/px_r$r.log 2>&1
done
timeout 900 ncu --set full --clock-control none -k regex:"k_poly|k_pass" -s 6 -c 6 -o gpurun_out/px_pc3_medium -f python tools/prof_solve.py medium 4 3 > gpurun_out/px_ncu.log 2>&1
python tools/ncu_summary.py gpurun_out/px_pc3_medium.ncu-rep > gpurun_out/px_ncu_summary.txt 2>&1
