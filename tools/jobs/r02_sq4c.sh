timeout 1500 python -m pytest tests -m gpu -q -rf > gpurun_out/r02_pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/r02_pytest_gpu.log
timeout 600 python tools/sq4_check.py > gpurun_out/r02_sq4.log 2>&1; echo "sq4 rc $?"; tail -6 gpurun_out/r02_sq4.log
timeout 600 python tools/horizon_sweep.py 8192 > gpurun_out/r02_horizon_sweep.json 2>/dev/null; python -c "import json; d=json.load(open('gpurun_out/r02_horizon_sweep.json'));[print(r['horizon'], r['ms_per_tick_p50'], r['roofline_frac']) for r in d['rows']]"
