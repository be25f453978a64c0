# attention schedule variants at C3: whole step (unprofiled ms/step) + profiled attention ms
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
for V in default tail sk st4 st6 st8; do
  unset FOCUS_ATTN_SK FOCUS_ATTN_TAIL FOCUS_ATTN_SPLIT_TILES
  case $V in tail) export FOCUS_ATTN_TAIL=1;; sk) export FOCUS_ATTN_SK=1;; st4) export FOCUS_ATTN_SPLIT_TILES=4;; st6) export FOCUS_ATTN_SPLIT_TILES=6;; st8) export FOCUS_ATTN_SPLIT_TILES=8;; esac
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$V.json 2> gpurun_out/bench_$V.err
  python -c "
import json; d=json.load(open('gpurun_out/bench_$V.json'))
print('$V', d['value'], d['ms_per_step'], d['kernels']['attention'], d['kernels']['gemm_qkv']['ms_per_step'])"
done
