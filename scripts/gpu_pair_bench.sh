python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -I include scripts/gemm_bench.cu -o /tmp/gemm_bench -Lpaper_2601_23278_b200 -lfocus -Xlinker -rpath=$PWD/paper_2601_23278_b200 2>/dev/null || exit 1
for M in 428 200; do
GEMM_TAG=sk GEMM_TRACE=1 FOCUS_GEMM_PSK=1 timeout 60 /tmp/gemm_bench $M | grep -v "check.*OK"
GEMM_TAG=dp FOCUS_GEMM_PSK=0 timeout 60 /tmp/gemm_bench $M | grep -v "check.*OK"
done
timeout 600 python -m pytest tests/test_gpu_layers.py -x -q -m gpu 2>&1 | tail -3
for P in 2 0; do
  if [ $P = 0 ]; then export FOCUS_GEMM_PSK=0; fi
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_psk$P.json 2> gpurun_out/bench.err; echo "bench rc $?"
  python -c "
import json; d=json.load(open('gpurun_out/bench_psk$P.json'))
print('psk$P', d['value'], d['ms_per_step'], {k:round(v['ms_per_step'],3) for k,v in d['kernels'].items() if k.startswith('gemm') or k.startswith('att')})"
done
