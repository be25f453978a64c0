# dynamic attention schedule: GPU tests, bench, attention trace
FOCUS_TEST_LOG=gpurun_out/r2_gemm_errors.jsonl timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/r2_dyn_pytest.log 2>&1; echo "pytest rc $?"
tail -5 gpurun_out/r2_dyn_pytest.log
timeout 900 python bench.py > gpurun_out/r2_dyn_bench.json 2> gpurun_out/r2_dyn_bench.err; echo "bench rc $?"
tail -3 gpurun_out/r2_dyn_bench.err
python - <<'PY'
import json
d=json.loads(open('gpurun_out/r2_dyn_bench.json').read().strip().splitlines()[-1])
print({k: d[k] for k in ('value','ms_per_step','generation','clocks')})
print([ (w['start'], w['value']) for w in d['windows']])
print('e2e', d['e2e']['value']); print('attn', d['kernels']['attention'])
print('none', d['no_eviction']['generation'], d['no_eviction'].get('focus_speedup_generation')); print('cal', d['calibrated'])
PY
timeout 300 python scripts/attn_trace.py 10 > /dev/null 2>&1; echo "trace rc $?"
python scripts/attn_trace_report.py gpurun_out/attn_trace.npz > gpurun_out/r2_dyn_attn_trace.txt 2>&1; tail -6 gpurun_out/r2_dyn_attn_trace.txt
