python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_layers.py -q -x 2>&1 | tail -1
for V in "0 0" "4 2" "8 2" "16 4" "8 0" "0 4"; do
  set -- $V
  FOCUS_GEMM_PF=$1 FOCUS_ATTN_PF=$2 timeout 300 python bench.py --steps 8 --warmup 3 --no-cpu-baseline > gpurun_out/bench_pf.json 2> gpurun_out/bench.err
  python -c "
import json; d=json.load(open('gpurun_out/bench_pf.json'))
print('gemm_pf=$1 attn_pf=$2', d['value'], d['ms_per_step'], {k:round(v['ms_per_step'],3) for k,v in d['kernels'].items() if k.startswith('gemm') or k=='attention'})"
done
