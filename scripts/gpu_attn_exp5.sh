python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 200 python scripts/attn_trace.py 10 > /dev/null 2>&1; python scripts/attn_trace_report.py gpurun_out/attn_trace.npz > gpurun_out/attn_trace_epi.txt 2>&1
grep -E "===|epilogue|MMA" gpurun_out/attn_trace_epi.txt
