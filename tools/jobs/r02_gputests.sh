timeout 1500 python -m pytest tests -m gpu -q -rf > gpurun_out/r02_pytest_gpu.log 2>&1; echo "pytest rc $?"
tail -5 gpurun_out/r02_pytest_gpu.log
timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool racecheck --racecheck-report all python tools/racecheck.py 2 10 > gpurun_out/r02_racecheck.log 2>&1; echo "racecheck rc $?"
tail -8 gpurun_out/r02_racecheck.log
