timeout 900 python -m pytest tests/test_gpu_soa.py tests/test_abi.py -q -rf -x > gpurun_out/r02_soa_tests.log 2>&1; echo "soa tests rc $?"; tail -4 gpurun_out/r02_soa_tests.log
timeout 600 python bench.py --no-ppo --cl-agents 0 --no-cpu-baseline > gpurun_out/r02_bench_soa.json 2> gpurun_out/r02_bench_soa.err; echo "bench rc $?"
python -c "import json; d=json.load(open('gpurun_out/r02_bench_soa.json')); print(d['value'], d['ms_per_step'], d['gpu_launches'], json.dumps(d['e2e']))"
