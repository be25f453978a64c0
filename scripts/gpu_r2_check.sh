# round-2 checks: new parity tests, graph replay, logit-scale calibration, bench
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_graph.py -m gpu -x -q -k "threshold or full_vocab or graph_replay" > gpurun_out/r2_check_pytest.log 2>&1; echo "pytest rc $?"
tail -15 gpurun_out/r2_check_pytest.log
timeout 600 python scripts/calibrate_logit_scale.py C3 16 34 > gpurun_out/r2_calib.log 2>&1; echo "calib rc $?"; cat gpurun_out/r2_calib.log | tail -8
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r2_check_bench.json 2> gpurun_out/r2_check_bench.err; echo "bench rc $?"
python -c "
import json;d=json.loads(open('gpurun_out/r2_check_bench.json').read().strip().splitlines()[-1]);print(d['value'],d['ms_per_step'],d['e2e']['value'],d['clocks'],d['roofline']['frac'])"
