timeout 1500 python -m pytest tests -m gpu -q -rf > gpurun_out/r02_pytest_gpu.log 2>&1; echo "tests rc $?"; tail -4 gpurun_out/r02_pytest_gpu.log
