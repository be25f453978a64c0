python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
# prefill launches: 64 requests x (1 embed + 36 layers x (rmsnorm, qkv, attn, o, rmsnorm, gu, down)) = 64 x 253 = 16192
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 16300 -c 700 --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo "ncu rc $?"
