# thin-slab study: per-rank 19 shells (medium at N=8) on 4 GPUs vs 1 GPU
T="timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29516"
timeout 300 python tools/lat.py 19x301x601 400 2>&1 | grep us/iter
timeout 300 python tools/lat.py 38x301x601 400 2>&1 | grep us/iter
timeout 300 python tools/lat.py medium 200 2>&1 | grep us/iter
$T tools/lat.py 76x301x601 400 2>&1 | grep us/iter
$T tools/lat.py medium 400 2>&1 | grep us/iter
$T tools/mg_prof.py medium 2>&1 | grep total
