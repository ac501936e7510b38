timeout 600 python tools/share_check.py > gpurun_out/r02_share.log 2>&1; echo "share rc $?"
cat gpurun_out/r02_share.log | tail -30
timeout 1500 python -m pytest tests -m gpu -q -rf -x > gpurun_out/r02_pytest_gpu.log 2>&1; echo "pytest rc $?"
tail -5 gpurun_out/r02_pytest_gpu.log
