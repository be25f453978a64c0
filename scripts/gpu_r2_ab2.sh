# A/B: dynamic attention schedule (pull near unit end) x fused RMSNorm (batched residual loads)
timeout 900 python -m pytest tests/test_gpu_layers.py -m gpu -x -q -k "test_layer_stages and not multicast and not single and not stream and not tail and not unplanned" > gpurun_out/r2_ab2_pytest.log 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/r2_ab2_pytest.log
summ() { python - "$1" <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[1], 'value', d['value'], 'gen', d['generation']['value'], 'e2e', d['e2e']['value'], 'clk', d['clocks'].get('sm_mhz'), [w['value'] for w in d['windows']])
k=d.get('kernels',{}); print('  attn', k.get('attention',{}).get('ms_per_step'), 'rms', k.get('rmsnorm',{}).get('ms_per_step'), 'o', k.get('gemm_o',{}).get('ms_per_step'), 'gu', k.get('gemm_gu',{}).get('ms_per_step'), 'down', k.get('gemm_down',{}).get('ms_per_step'), 'qkv', k.get('gemm_qkv',{}).get('ms_per_step'))
PY
}
for cfg in "FOCUS_ATTN_DYN=1 FOCUS_FUSED_NORM=1" "FOCUS_ATTN_DYN=0 FOCUS_FUSED_NORM=1" "FOCUS_ATTN_DYN=1 FOCUS_FUSED_NORM=0" "FOCUS_ATTN_DYN=0 FOCUS_FUSED_NORM=0"; do
  echo "== $cfg"
  env $cfg timeout 600 python bench.py --no-extras --no-cpu-baseline > gpurun_out/r2_ab2.json 2>/dev/null; summ gpurun_out/r2_ab2.json
done
timeout 300 python scripts/attn_trace.py 10 > /dev/null 2>&1; python scripts/attn_trace_report.py gpurun_out/attn_trace.npz > gpurun_out/r2_ab2_trace_dyn.txt 2>&1; tail -4 gpurun_out/r2_ab2_trace_dyn.txt
FOCUS_ATTN_DYN=0 timeout 300 python scripts/attn_trace.py 10 > /dev/null 2>&1; python scripts/attn_trace_report.py gpurun_out/attn_trace.npz > gpurun_out/r2_ab2_trace_static.txt 2>&1; tail -4 gpurun_out/r2_ab2_trace_static.txt
