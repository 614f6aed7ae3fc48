# ncu --set full of pass A and pass B (even iterations) on the large grid
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_pass_a|k_pass_b_pc1_even" -s 4 -c 2 -o gpurun_out/passes_large -f python tools/prof_solve.py large 8 > gpurun_out/ncu_passes.log 2>&1
python tools/ncu_summary.py gpurun_out/passes_large.ncu-rep > gpurun_out/ncu_passes_summary.txt 2>&1
