python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -2 gpurun_out/pytest_gpu.log
for V in plan sk noplan; do
  unset FOCUS_ATTN_SK FOCUS_ATTN_NOPLAN
  if [ $V = sk ]; then export FOCUS_ATTN_SK=1; fi
  if [ $V = noplan ]; then export FOCUS_ATTN_NOPLAN=1; fi
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$V.json 2> gpurun_out/bench.err; echo "bench rc $?"
  python -c "
import json; d=json.load(open('gpurun_out/bench_$V.json'))
print('$V', d['value'], d['ms_per_step'], d['kernels']['attention'])"
done
