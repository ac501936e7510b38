timeout 1500 python -m pytest tests -m gpu -q -rf > gpurun_out/r02_pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -4 gpurun_out/r02_pytest_gpu.log
timeout 900 python tools/ref_parity.py gpurun_out/r02_ref_parity.json > gpurun_out/r02_ref_parity.log 2>&1; echo "ref_parity rc $?"
timeout 900 python tools/configs.py > gpurun_out/r02_configs.json 2> gpurun_out/r02_configs.err; echo "configs rc $?"; cat gpurun_out/r02_configs.err | tail -8
