cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sweepS -s 2 -c 2 -o gpurun_out/g12_sweepS_medium -f python tools/prof_solve.py medium 4 2 > gpurun_out/g12_ncu.log 2>&1
python tools/ncu_summary.py gpurun_out/g12_sweepS_medium.ncu-rep > gpurun_out/g12_ncu_summary.txt 2>&1
python tools/ncu_sass_hot.py gpurun_out/g12_sweepS_medium.ncu-rep k_sweepS 30 4 > gpurun_out/g12_hot.txt 2>&1
