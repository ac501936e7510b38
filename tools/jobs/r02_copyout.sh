timeout 1500 python -m pytest tests -m gpu -q -rf -x > gpurun_out/r02_pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -4 gpurun_out/r02_pytest_gpu.log
timeout 600 python bench.py --no-ppo --cl-agents 0 --no-cpu-baseline > gpurun_out/r02_bench_co.json 2> gpurun_out/r02_bench_co.err; echo "bench rc $?"
python -c "import json; d=json.load(open('gpurun_out/r02_bench_co.json')); print(d['value'], d['ms_per_step'], d['gpu_launches'], json.dumps(d['e2e']))"
timeout 300 python tools/latency_split.py 10 2>&1 | tail -4
