timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_soa.py -q -rf -x > gpurun_out/r02_pytest_co2.log 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/r02_pytest_co2.log
timeout 600 python bench.py --no-ppo --cl-agents 0 --no-cpu-baseline > gpurun_out/r02_bench_co2.json 2> gpurun_out/r02_bench_co2.err; echo "bench rc $?"
python -c "import json; d=json.load(open('gpurun_out/r02_bench_co2.json')); print(d['value'], d['ms_per_step'], d['gpu_launches'], json.dumps(d['e2e']))"
