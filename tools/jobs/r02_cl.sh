timeout 900 python -m pytest tests/test_gpu_closed_loop.py tests/test_gpu_parity.py -k "closed_loop or sharing" -m gpu -q -rf -s > gpurun_out/r02_closed_loop.log 2>&1; echo "pytest rc $?"
grep -E "substeps|passed|failed" gpurun_out/r02_closed_loop.log
timeout 600 python tools/time_solve.py 16384 5 10 20
timeout 600 python bench.py --no-ppo --cl-agents 0 --no-cpu-baseline > gpurun_out/r02_bench2.json 2>&1; echo "bench rc $?"
python -c "import json; d=json.load(open('gpurun_out/r02_bench2.json')); print(d['value'], d['ms_per_step'], d['e2e']['ms_per_step'], d['e2e']['last_timing_ms'], d['e2e']['without_z_star'])"
