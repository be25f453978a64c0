python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/pytest_gpu.log
for P in tail notail; do
  if [ $P = notail ]; then export FOCUS_ATTN_NOTAIL=1; fi
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$P.json 2> gpurun_out/bench.err; echo "bench rc $?"
  python -c "
import json; d=json.load(open('gpurun_out/bench_$P.json'))
print('$P', d['value'], d['ms_per_step'], {k:round(v['ms_per_step'],3) for k,v in d['kernels'].items() if k.startswith('gemm') or k.startswith('att')})"
done
unset FOCUS_ATTN_NOTAIL
timeout 200 python scripts/attn_trace.py 10 2>&1 | tail -1
