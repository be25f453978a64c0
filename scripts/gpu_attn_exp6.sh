python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
for V in default tail sk st8; do
  unset FOCUS_ATTN_SK FOCUS_ATTN_TAIL FOCUS_ATTN_SPLIT_TILES
  case $V in tail) export FOCUS_ATTN_TAIL=1;; sk) export FOCUS_ATTN_SK=1;; st8) export FOCUS_ATTN_SPLIT_TILES=8;; esac
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$V.json 2> gpurun_out/bench_$V.err
  python -c "
import json; d=json.load(open('gpurun_out/bench_$V.json'))
print('$V', d['value'], d['ms_per_step'], d['kernels']['attention'])"
  timeout 200 python scripts/attn_trace.py 10 > /dev/null 2>&1; python scripts/attn_trace_report.py gpurun_out/attn_trace.npz > gpurun_out/attn_trace_$V.txt 2>&1
  grep -E "epilogue  0|CTA span" gpurun_out/attn_trace_$V.txt
done
