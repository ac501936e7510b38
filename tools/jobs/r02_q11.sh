timeout 1500 python -m pytest tests -m gpu -q -rf -x > gpurun_out/r02_pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -2 gpurun_out/r02_pytest_gpu.log
timeout 900 python tools/paths.py > gpurun_out/r02_paths.jsonl 2> gpurun_out/r02_paths.err; echo "paths rc $?"; cat gpurun_out/r02_paths.jsonl | cut -c1-140
python tools/latency_split.py 10 2>&1 | tail -3
