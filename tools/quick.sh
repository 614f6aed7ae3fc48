# quick GPU check: parity tests + bench N=1 (no cpu baseline)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/q_tests.log 2>&1; echo "tests rc $?"; tail -3 gpurun_out/q_tests.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/q_bench.log 2>&1; echo "bench rc $?"
python - <<'PY'
import json
d=json.loads(open('gpurun_out/q_bench.log').read().strip().splitlines()[-1])
r=d['roofline']
print('value', round(d['value'],1), 'ms/step', round(d['ms_per_step'],1), 'passA', r['pass_a'], 'passB', r['pass_b'], 'e2e', round(d['e2e']['value'],1))
PY
