# full GPU test suite + the default bench (and a C2 line)
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/r2_pytest.log 2>&1; echo "pytest rc $?"
tail -5 gpurun_out/r2_pytest.log
timeout 900 python bench.py > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err; echo "bench rc $?"
tail -5 gpurun_out/r2_bench.err
python - <<'PY'
import json
d=json.loads(open('gpurun_out/r2_bench.json').read().strip().splitlines()[-1])
print({k: d[k] for k in ('value','ms_per_step','windows','generation','redundancy','clocks','gpu_launches')})
print('e2e', d['e2e']); print('roof', d.get('roofline')); print('step', d.get('step_roofline'))
print('none', d.get('no_eviction')); print('cal', d.get('calibrated'))
PY
