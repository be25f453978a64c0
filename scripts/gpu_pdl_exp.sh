python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -2 gpurun_out/pytest_gpu.log
for V in 1 0 1; do
  FOCUS_PDL=$V timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_pdl$V.json 2> gpurun_out/bench.err; echo "bench rc $?"
  python -c "
import json; d=json.load(open('gpurun_out/bench_pdl$V.json'))
print('pdl=$V', d['value'], d['ms_per_step'], d['e2e']['value'], d['clocks'])"
done
