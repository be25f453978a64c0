#!/bin/bash
# GPU evidence suite (run on a B200 box via gpurun; outputs under gpurun_out/, summaries go to profiles/).
#   bash scripts/gpu_suite.sh tests      -- pytest -m gpu
#   bash scripts/gpu_suite.sh bench      -- default bench line (C3, whole generation)
#   bash scripts/gpu_suite.sh launches   -- ncu launch list (gpu__time_duration) of one mid-generation C3 step
#   bash scripts/gpu_suite.sh full       -- ncu --set full of layer 10's kernels of one mid-generation step
#   bash scripts/gpu_suite.sh small      -- ncu DRAM metrics of the FOCUS bookkeeping kernels (select, gather,
#                                           vocab reduce, commit, setup, embed, rmsnorm, plan) of one step
#   bash scripts/gpu_suite.sh sanitize   -- compute-sanitizer memcheck / racecheck / synccheck on smoke()
mkdir -p gpurun_out
case "$1" in
  tests) timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/pytest_gpu.log ;;
  bench) timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc $?"; tail -c 400 gpurun_out/bench.json ;;
  launches)
    timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/launches_mid.csv python scripts/profile_step.py C3 260 > gpurun_out/launches_mid.log 2>&1
    echo "ncu rc $?" ;;
  full)
    # one mid-generation step: layer-10 kernels = launches 11*6.. of the step (QKV, attention, O, GU, down)
    timeout 1500 ncu --profile-from-start off --set full --clock-control none --import-source on \
      -k regex:"k_gemm_pair|k_attn_tc" -s 61 -c 5 -o gpurun_out/full_mid python scripts/profile_step.py C3 260 \
      > gpurun_out/full_mid.log 2>&1; echo "ncu rc $?"
    python scripts/ncu_summary.py gpurun_out/full_mid.ncu-rep > gpurun_out/full_mid_summary.txt 2>&1 ;;
  small)
    timeout 900 ncu --profile-from-start off --clock-control none --csv \
      --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum \
      -k regex:"k_select_plan|k_gather_rows|k_vocab_reduce|k_commit|k_step_setup|k_embed|k_rmsnorm|k_attn_plan|k_rope_rows" \
      --log-file gpurun_out/small_kernels.csv python scripts/profile_step.py C3 260 > gpurun_out/small.log 2>&1
    echo "ncu rc $?" ;;
  sanitize)
    for tool in memcheck racecheck synccheck; do
      timeout 1200 compute-sanitizer --tool $tool --print-limit 20 python -c "import __graft_entry__ as g; g.smoke()" \
        > gpurun_out/sanitize_$tool.log 2>&1; echo "$tool rc $?"; tail -3 gpurun_out/sanitize_$tool.log
    done ;;
esac
