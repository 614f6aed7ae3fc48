T="timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
POT3D_EDGE_IN_A=1 $T --master-port 29571 tools/mgpu_check.py 2>&1 | grep -E " OK | FAIL" | cut -c1-120
for f in 0 1 0 1; do
  POT3D_EDGE_IN_A=$f $T --master-port 2957$((2+f)) tools/lat.py 76x301x601 400 2>&1 | grep us/iter | sed "s/^/edgeA=$f /"
  POT3D_EDGE_IN_A=$f $T --master-port 2957$((4+f)) tools/lat.py medium 400 2>&1 | grep us/iter | sed "s/^/edgeA=$f /"
done
