set -x
timeout 900 python tools/ref_parity.py gpurun_out/r02_ref_parity.json > gpurun_out/r02_ref_parity.log 2>&1; echo "ref_parity rc $?"
timeout 900 python -m pytest tests/test_gpu_ref_parity.py tests/test_gpu_parity.py -m gpu -q -rf -s > gpurun_out/r02_pytest_parity.log 2>&1; echo "pytest rc $?"
