python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
for V in default tail; do
  unset FOCUS_ATTN_TAIL; case $V in tail) export FOCUS_ATTN_TAIL=1;; esac
  timeout 200 python scripts/attn_trace.py 10 > /dev/null 2>&1; python scripts/attn_trace_report.py gpurun_out/attn_trace.npz > gpurun_out/attn_trace_$V.txt 2>&1
  echo $V; tail -5 gpurun_out/attn_trace_$V.txt
done
