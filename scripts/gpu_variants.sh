# usage: bash scripts/gpu_variants.sh "name:ENV=V,ENV=V" ...   (C3 bench per variant, unprofiled ms/step + kernels)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
for spec in "$@"; do
  name=${spec%%:*}; envs=${spec#*:}
  ( IFS=','; for kv in $envs; do [ -n "$kv" ] && export "$kv"; done
    timeout 300 python bench.py --steps ${STEPS:-10} --warmup 3 --no-cpu-baseline > gpurun_out/bench_$name.json 2> gpurun_out/bench_$name.err
    python -c "
import json; d=json.load(open('gpurun_out/bench_$name.json')); k=d['kernels']
print('%-10s %8.1f tok/s %7.3f ms  e2e %7.1f | ' % ('$name', d['value'], d['ms_per_step'], d['e2e']['value']) + ' '.join('%s=%.3f' % (n[:8], v['ms_per_step']) for n, v in k.items() if v['ms_per_step'] > 0.05))" )
done
