# layer-10 attention launch: global-time span (entry -> last exit) over 3 traced runs
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
for i in 1 2 3; do
  timeout 200 python scripts/attn_trace.py 10 > /dev/null 2>&1; python scripts/attn_trace_report.py gpurun_out/attn_trace.npz 2>&1 | grep -E "global time|CTA span"
done
