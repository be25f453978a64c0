python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 300 python -m pytest tests/test_gpu_layers.py -x -q 2>&1 | tail -3
for ST in 16 4; do
  FOCUS_ATTN_SPLIT_TILES=$ST timeout 200 python scripts/attn_trace.py 10 > /dev/null 2>&1; echo "trace rc $?"
  cp gpurun_out/attn_trace.npz gpurun_out/attn_trace_st$ST.npz
  FOCUS_ATTN_SPLIT_TILES=$ST timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_st$ST.json 2> gpurun_out/bench.err; echo "bench rc $?"
  python -c "
import json; d=json.load(open('gpurun_out/bench_st$ST.json'))
print('ST=$ST', d['value'], d['ms_per_step'], d['kernels']['attention'])"
done
