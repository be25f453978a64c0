# A/B of one kernel family's device time over one decode step under ncu (clock-control base: stable
# clocks for comparisons; not a bench number).  usage: gpu_ab_kernel.sh REGEX "name:ENV=V,..." ...
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
re=$1; shift
for spec in "$@"; do
  name=${spec%%:*}; envs=${spec#*:}
  ( IFS=','; for kv in $envs; do [ -n "$kv" ] && export "$kv"; done
    FOCUS_NCU_STEP=1 timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum -k regex:"$re" --csv --log-file gpurun_out/ab_$name.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
    python - "$name" <<'PY'
import csv, sys
name = sys.argv[1]
rows = [r for r in csv.reader(open(f"gpurun_out/ab_{name}.csv")) if len(r) > 5]
h = rows[0]; iv = h.index("Metric Value"); ik = h.index("Kernel Name")
v = [float(r[iv].replace(",", "")) for r in rows[1:]]
print(f"{name:10s} launches {len(v):3d} total {sum(v)/1e3:8.1f} us  mean {sum(v)/max(1,len(v))/1e3:7.2f} us")
PY
  )
done
