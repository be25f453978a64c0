# attention: I-cache footprint experiment (one softmax variant) + traces
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
for V in default nch4; do
  unset FOCUS_ATTN_NCH4
  case $V in nch4) export FOCUS_ATTN_NCH4=1;; esac
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$V.json 2> gpurun_out/bench_$V.err
  python -c "
import json; d=json.load(open('gpurun_out/bench_$V.json'))
print('$V', d['value'], d['ms_per_step'], d['kernels']['attention'])"
  timeout 200 python scripts/attn_trace.py 10 > /dev/null 2>&1; python scripts/attn_trace_report.py gpurun_out/attn_trace.npz > gpurun_out/attn_trace_$V.txt 2>&1
  tail -12 gpurun_out/attn_trace_$V.txt
done
