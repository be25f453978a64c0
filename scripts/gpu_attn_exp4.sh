python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
for V in tail st8; do
  unset FOCUS_ATTN_TAIL FOCUS_ATTN_SPLIT_TILES
  case $V in tail) export FOCUS_ATTN_TAIL=1;; st8) export FOCUS_ATTN_SPLIT_TILES=8;; esac
  timeout 200 python scripts/attn_trace.py 10 > /dev/null 2>&1; python scripts/attn_trace_report.py gpurun_out/attn_trace.npz > gpurun_out/attn_trace_$V.txt 2>&1
  cp gpurun_out/attn_trace.npz gpurun_out/attn_trace_$V.npz
  tail -22 gpurun_out/attn_trace_$V.txt
done
