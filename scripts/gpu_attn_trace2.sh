python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
FOCUS_ATTN_SK=1 timeout 200 python scripts/attn_trace.py 10 2>&1 | tail -2; echo "trace rc $?"
