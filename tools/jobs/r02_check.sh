set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
nproc; lscpu | grep "Model name"
timeout 1500 python -m pytest tests -m gpu -q -rf > gpurun_out/r02_pytest_gpu.log 2>&1; echo "pytest rc $?"
tail -30 gpurun_out/r02_pytest_gpu.log
timeout 900 python tools/ref_parity.py gpurun_out/r02_ref_parity.json > gpurun_out/r02_ref_parity.log 2>&1; echo "ref_parity rc $?"
timeout 600 python bench.py > gpurun_out/r02_bench.json 2> gpurun_out/r02_bench.err; echo "bench rc $?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r02_bench_ref.json 2> gpurun_out/r02_bench_ref.err; echo "ref rc $?"
