cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for ca in 0 6 8 12; do
  if [ $ca = 0 ]; then unset POT3D_CHUNKS; else export POT3D_CHUNKS=$ca; fi
  timeout 300 python tools/pass_times.py large 300 >> gpurun_out/g8_chunks.log 2>&1
done
unset POT3D_CHUNKS
for cb in 6 16; do
  POT3D_CHUNKS_B=$cb timeout 300 python tools/pass_times.py large 300 >> gpurun_out/g8_chunks.log 2>&1
done
timeout 300 python tools/pass_times.py large 300 1 >> gpurun_out/g8_chunks.log 2>&1
timeout 300 python tools/pass_times.py medium 600 >> gpurun_out/g8_chunks.log 2>&1
timeout 300 python tools/pass_times.py medium 600 1 >> gpurun_out/g8_chunks.log 2>&1
