# A/B of the dynamic attention schedule and the fused RMSNorm; full GPU tests first
FOCUS_TEST_LOG=gpurun_out/r2_gemm_errors.jsonl timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/r2_ab_pytest.log 2>&1; echo "pytest rc $?"
tail -5 gpurun_out/r2_ab_pytest.log
summ() { python - "$1" <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[1], 'value', d['value'], 'gen', d['generation']['value'], 'e2e', d['e2e']['value'], 'clk', d['clocks'].get('sm_mhz'), [w['value'] for w in d['windows']])
k=d.get('kernels',{}); print('  attn', k.get('attention',{}).get('ms_per_step'), 'rms', k.get('rmsnorm',{}).get('ms_per_step'), 'o', k.get('gemm_o',{}).get('ms_per_step'), 'gu', k.get('gemm_gu',{}).get('ms_per_step'), 'down', k.get('gemm_down',{}).get('ms_per_step'), 'qkv', k.get('gemm_qkv',{}).get('ms_per_step'))
for x in ('no_eviction','calibrated'):
    if x in d: print(' ', x, d[x]['generation']['value'], d[x].get('focus_speedup_generation'), d[x].get('decoded_per_request_step'))
PY
}
timeout 900 python bench.py > gpurun_out/r2_ab_default.json 2> gpurun_out/r2_ab_default.err; echo "bench rc $?"; summ gpurun_out/r2_ab_default.json
FOCUS_ATTN_DYN=0 timeout 600 python bench.py --no-extras --no-cpu-baseline > gpurun_out/r2_ab_static.json 2>/dev/null; summ gpurun_out/r2_ab_static.json
FOCUS_FUSED_NORM=0 timeout 600 python bench.py --no-extras --no-cpu-baseline > gpurun_out/r2_ab_nofuse.json 2>/dev/null; summ gpurun_out/r2_ab_nofuse.json
timeout 300 python scripts/attn_trace.py 10 > /dev/null 2>&1; python scripts/attn_trace_report.py gpurun_out/attn_trace.npz > gpurun_out/r2_ab_trace_dyn.txt 2>&1; tail -4 gpurun_out/r2_ab_trace_dyn.txt
