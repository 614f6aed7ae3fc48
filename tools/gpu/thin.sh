# Thin r-slabs (the per-GPU slab of large on 8 GPUs: 38 shells x 601 x 1201) on 4 GPUs: chunking of
# the fused passes and the edge-shell dispatch (A/B knobs), against the same grid on 1 GPU
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
R4="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
B="bench.py --config large8slab --steps 2 --warmup 2 --no-cpu-baseline"
timeout 900 $R4 --master-port 29639 tools/mgpu_check.py > gpurun_out/t8_check_peer.log 2>&1; echo rc=$? >> gpurun_out/t8_check_peer.log
timeout 900 python $B > gpurun_out/t8_n1.log 2>&1
port=29640
for v in default mina2 mina1 chunks4 chunksb1 chunksb3 edgek; do
  unset POT3D_MIN_CHUNKS_A POT3D_CHUNKS POT3D_CHUNKS_B POT3D_EDGE_IN_A
  case $v in
    mina2) export POT3D_MIN_CHUNKS_A=2;;
    mina1) export POT3D_MIN_CHUNKS_A=1 POT3D_CHUNKS=1;;
    chunks4) export POT3D_CHUNKS=4;;
    chunksb1) export POT3D_CHUNKS_B=1;;
    chunksb3) export POT3D_CHUNKS_B=3;;
    edgek) export POT3D_EDGE_IN_A=0;;
  esac
  port=$((port+1))
  timeout 900 $R4 --master-port $port $B --gpus 4 > gpurun_out/t8_n4_$v.log 2>&1
done
