timeout 1500 python -m pytest tests -m gpu -q -rf -x > gpurun_out/r02_pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/r02_pytest_gpu.log
timeout 600 python bench.py --no-ppo --no-cpu-baseline --cl-agents 0 > gpurun_out/r02_q16_bench.json 2>gpurun_out/r02_q16_bench.err; echo "bench rc $?"
python -c "import json; d=json.load(open('gpurun_out/r02_q16_bench.json')); print(d['value'], d['ms_per_step'], d['e2e']['value'], d['e2e']['ms_per_step'], d['e2e']['last_timing_ms'], d['e2e']['without_z_star'], d['e2e']['soa']['ms_per_step'])"
