# squad kernel: the GPU test suite and the bench line
timeout 1500 python -m pytest tests -m gpu -q -rf -x > gpurun_out/r02_pytest_gpu.log 2>&1; echo "pytest rc $?"
tail -15 gpurun_out/r02_pytest_gpu.log
timeout 600 python bench.py > gpurun_out/r02_bench.json 2> gpurun_out/r02_bench.err; echo "bench rc $?"
python -c "import json; d=json.load(open('gpurun_out/r02_bench.json')); print(d['value'], d['ms_per_step'], d['e2e']['value'], d['e2e']['ms_per_step'], d['roofline']['frac'], d['closed_loop']['p50_tick_ms'])"
