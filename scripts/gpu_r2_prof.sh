# ncu launch list of one mid-generation C3 step + a clock64 trace of a layer-10 attention launch
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches_mid.csv python scripts/profile_step.py C3 260 > gpurun_out/r2_prof_step.log 2>&1; echo "ncu rc $?"
tail -2 gpurun_out/r2_prof_step.log
timeout 300 python scripts/attn_trace.py 10 > /dev/null 2>&1; echo "trace rc $?"
python scripts/attn_trace_report.py gpurun_out/attn_trace.npz > gpurun_out/r2_attn_trace.txt 2>&1; tail -12 gpurun_out/r2_attn_trace.txt
