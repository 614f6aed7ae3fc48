T="timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
POT3D_XFER_FORK=1 $T --master-port 29541 tools/mgpu_check.py 2>&1 | grep -cE " OK "
for f in 0 1 0 1; do
  POT3D_XFER_FORK=$f $T --master-port 2954$((2+f)) tools/lat.py 76x301x601 400 2>&1 | grep us/iter | sed "s/^/fork=$f /"
  POT3D_XFER_FORK=$f $T --master-port 2954$((4+f)) tools/lat.py medium 400 2>&1 | grep us/iter | sed "s/^/fork=$f /"
done
