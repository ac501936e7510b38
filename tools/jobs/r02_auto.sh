timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_soa.py tests/test_gpu_determinism.py -q -rf > gpurun_out/r02_auto_tests.log 2>&1; echo "tests rc $?"; tail -4 gpurun_out/r02_auto_tests.log
timeout 900 python tools/configs.py > gpurun_out/r02_configs.json 2> gpurun_out/r02_configs.err; echo "configs rc $?"; cat gpurun_out/r02_configs.err | tail -8
