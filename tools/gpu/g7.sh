# ncu of the FAST passes on large; compute-sanitizer on the protocols
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_pass_a|k_pass_b_pc1_even" -s 4 -c 2 -o gpurun_out/g7_passes_large -f python tools/prof_solve.py large 8 > gpurun_out/g7_ncu.log 2>&1
python tools/ncu_summary.py gpurun_out/g7_passes_large.ncu-rep > gpurun_out/g7_ncu_summary.txt 2>&1
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_cases.py > gpurun_out/g7_san_$tool.log 2>&1; echo "rc=$?" >> gpurun_out/g7_san_$tool.log
done
