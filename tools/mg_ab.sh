# multi-GPU: parity check + bench A/B of PDL: tools/mg_ab.sh N
N=${1:-2}
mkdir -p gpurun_out
T="timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511"
$T tools/mgpu_check.py > gpurun_out/mg${N}_check.log 2>&1; echo "check rc $?"; grep "ranks\]" gpurun_out/mg${N}_check.log
for pdl in 0 1; do
POT3D_PDL=$pdl $T bench.py --gpus $N --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/mg${N}_bench_pdl$pdl.log 2>&1
python - gpurun_out/mg${N}_bench_pdl$pdl.log $pdl <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(f"N={d['n_gpus']} PDL={sys.argv[2]} value {d['value']:.1f} {d['unit']} ms/step {d['ms_per_step']:.1f}")
PY
done
