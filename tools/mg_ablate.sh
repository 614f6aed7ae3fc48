T="timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29519"
for env in "X=0" "POT3D_PDL=0" "POT3D_XFER=0" "POT3D_EDGE_BLOCKS=148" "POT3D_EDGE_BLOCKS=296" "POT3D_EDGE_BLOCKS=1184"; do
  env $env $T tools/lat.py 76x301x601 400 2>&1 | grep us/iter | sed "s/^/$env /"
done
