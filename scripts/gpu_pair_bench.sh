python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -I include scripts/gemm_bench.cu -o /tmp/gemm_bench -Lpaper_2601_23278_b200 -lfocus -Xlinker -rpath=$PWD/paper_2601_23278_b200 2>/dev/null || exit 1
GEMM_TAG=pair FOCUS_GEMM_PAIR=1 timeout 60 /tmp/gemm_bench 428 | grep -v check
for P in pair1 pair0; do
  export FOCUS_GEMM_PAIR=${P#pair}
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$P.json 2> gpurun_out/bench.err; echo "bench rc $?"
  python -c "
import json; d=json.load(open('gpurun_out/bench_$P.json'))
print('$P', d['value'], d['ms_per_step'], {k:round(v['ms_per_step'],3) for k,v in d['kernels'].items() if k.startswith('gemm') or k=='attention'})"
done
FOCUS_GEMM_PAIR=1 timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest(pair) rc $?"; tail -2 gpurun_out/pytest_gpu.log
