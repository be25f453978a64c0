set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 300 python -m pytest tests/test_gpu_layers.py -x -q 2>&1 | tail -5
timeout 200 python scripts/attn_trace.py 10 > /dev/null 2>&1; echo "trace rc $?"
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc $?"
head -c 3000 gpurun_out/bench.json; tail -3 gpurun_out/bench.err
